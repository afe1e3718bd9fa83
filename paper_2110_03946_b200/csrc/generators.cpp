// Seeded input generators of the reference, behind the C ABI.
//
// synthetic_test_image (synthetic.hpp:14-59): per channel, five Gaussian
// blobs over a low-frequency sinusoid product, rescaled into [0.05, 0.95].
// random_mask (masks.hpp:25-43): exactly llround(density*N) known pixels by
// a partial Fisher-Yates shuffle of the pixel indices.
//
// Both draw from std::mt19937_64 through libstdc++'s distributions in the
// reference's draw order, so the bytes match the reference's on the same
// toolchain; the benchmark and parity tests feed identical inputs to the
// CPU reference and to the GPU path.  Host-only code (no device).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

#include "../../include/schwarz_b200.h"

extern "C" {

si_status si_synthetic_test_image(int w, int h, int c, uint64_t seed, double* out) {
  if (w <= 0 || h <= 0 || c <= 0 || !out) return SI_ERR_INVALID_ARGUMENT;
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  const double pi = 3.14159265358979323846;
  const double diag = std::sqrt(static_cast<double>(w) * w + static_cast<double>(h) * h);
  const size_t n = static_cast<size_t>(w) * h;
  struct Blob {
    double cx, cy, k, amp;  // centre, 1/(2 sigma^2), amplitude
  };
  for (int ch = 0; ch < c; ++ch) {
    Blob blobs[5];
    for (Blob& bl : blobs) {
      bl.cx = unit(gen) * w;
      bl.cy = unit(gen) * h;
      const double sigma = (0.05 + 0.20 * unit(gen)) * diag;
      bl.k = 1.0 / (2.0 * sigma * sigma);
      bl.amp = 0.3 + 0.7 * unit(gen);
    }
    const double fx = (1.0 + 2.0 * unit(gen)) * 2.0 * pi / w;
    const double fy = (1.0 + 2.0 * unit(gen)) * 2.0 * pi / h;
    const double phx = unit(gen) * 6.28318530717958647692;
    const double phy = unit(gen) * 6.28318530717958647692;
    double* plane = out + static_cast<size_t>(ch) * n;
    double lo = 1e300, hi = -1e300;
    for (int y = 0; y < h; ++y) {
      for (int x = 0; x < w; ++x) {
        double v = 0.4 * std::sin(fx * x + phx) * std::sin(fy * y + phy);
        for (const Blob& bl : blobs) {
          const double dx = x - bl.cx, dy = y - bl.cy;
          v += bl.amp * std::exp(-(dx * dx + dy * dy) * bl.k);
        }
        plane[static_cast<size_t>(y) * w + x] = v;
        lo = std::min(lo, v);
        hi = std::max(hi, v);
      }
    }
    const double scale = hi > lo ? 0.9 / (hi - lo) : 0.0;
    for (size_t i = 0; i < n; ++i) plane[i] = 0.05 + (plane[i] - lo) * scale;
  }
  return SI_OK;
}

si_status si_random_mask(int w, int h, double density, uint64_t seed, uint8_t* out) {
  if (w <= 0 || h <= 0 || !out || !(density > 0.0 && density <= 1.0))
    return SI_ERR_INVALID_ARGUMENT;
  const size_t n = static_cast<size_t>(w) * h;
  size_t k = static_cast<size_t>(std::llround(density * static_cast<double>(n)));
  k = std::min(k, n);
  if (k < 1) return SI_ERR_INVALID_ARGUMENT;
  std::vector<uint32_t> perm(n);
  std::iota(perm.begin(), perm.end(), 0u);
  std::fill(out, out + n, uint8_t{0});
  std::mt19937_64 gen(seed);
  for (size_t i = 0; i < k; ++i) {
    std::uniform_int_distribution<size_t> pick(i, n - 1);
    std::swap(perm[i], perm[pick(gen)]);
    out[perm[i]] = 1;
  }
  return SI_OK;
}

}  // extern "C"
