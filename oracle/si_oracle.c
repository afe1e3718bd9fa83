/* TEST INFRASTRUCTURE ONLY — the CPU parity oracle (see si_oracle.h).
 *
 * Plain C restatement of the reference's ORAS / multilevel-ORAS path.  The
 * arithmetic follows the reference's expression order so that, compiled with
 * the same contraction rules (gcc, -ffp-contract=fast), results agree with
 * the reference bit for bit; tests/test_oracle.py checks exactly that.
 * Citations are to /root/reference/proj/include/schwarz_inpaint/.
 */
#include "si_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

void or_default_options(or_options* o) {
  /* methods.hpp:40-55, schwarz.hpp:34,43-44 */
  o->tolerance = 1e-3;
  o->levels = 3;
  o->block_size = 32;
  o->overlap = 6;
  o->alpha = 0.25;
  o->coarse_tolerance = 1e-2;
  o->averaging = 0;
  o->local_tolerance = 1e-2;
  o->local_max_iterations = 30;
  o->local_check_interval = 30;
  o->max_outer_iterations = 1000;
  o->normalizer = 0;
  o->flavour = 1;
  o->cg_max_iterations = 100000;
  o->cg_check_interval = 4;
}

/* ---- deterministic sums: parallel.hpp:165-211 ------------------------- */
#define SUM_CHUNK 2048

/* lane_sum (parallel.hpp:172-189): eight accumulators chosen by the offset
 * from the range start, combined as a fixed pairwise tree. */
static double lane_dot(const double* a, const double* b, size_t begin, size_t end) {
  double lane[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  size_t i = begin;
  for (; i + 8 <= end; i += 8) {
    for (int k = 0; k < 8; ++k) lane[k] += a[i + k] * b[i + k];
  }
  for (int k = 0; i < end; ++i, ++k) lane[k] += a[i] * b[i];
  return ((lane[0] + lane[1]) + (lane[2] + lane[3])) + ((lane[4] + lane[5]) + (lane[6] + lane[7]));
}

/* parallel_sum of a[i]*b[i] (parallel.hpp:195-211; vec::dot cg.hpp:46-48). */
static double det_dot(const double* a, const double* b, size_t n) {
  if (n == 0) return 0.0;
  size_t chunks = (n + SUM_CHUNK - 1) / SUM_CHUNK;
  if (chunks == 1) return lane_dot(a, b, 0, n);
  double total = 0.0;
  for (size_t c = 0; c < chunks; ++c) {
    size_t begin = c * SUM_CHUNK;
    size_t end = begin + SUM_CHUNK < n ? begin + SUM_CHUNK : n;
    total += lane_dot(a, b, begin, end);
  }
  return total;
}

static double det_norm(const double* a, size_t n) { return sqrt(det_dot(a, a, n)); }

/* ---- global operator: operators.hpp:38-66, 81-97 ----------------------- */
static void op_apply(const uint8_t* mask, int w, int h, const double* u, double* out) {
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      size_t i = (size_t)y * w + x;
      if (mask[i]) {
        out[i] = u[i];
        continue;
      }
      double sum = 0.0;
      int deg = 0;
      if (x > 0) { sum += u[i - 1]; ++deg; }
      if (x + 1 < w) { sum += u[i + 1]; ++deg; }
      if (y > 0) { sum += u[i - w]; ++deg; }
      if (y + 1 < h) { sum += u[i + w]; ++deg; }
      out[i] = deg * u[i] - sum;
    }
  }
}

/* residual_into: r = b - A u (operators.hpp:91-97). */
static void residual_into(const uint8_t* mask, int w, int h, const double* u, const double* b,
                          double* r) {
  size_t n = (size_t)w * h;
  op_apply(mask, w, h, u, r);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
}

double or_residual_sumsq(const uint8_t* mask, int w, int h, const double* u, const double* b) {
  size_t n = (size_t)w * h;
  double* r = (double*)malloc(n * sizeof(double));
  residual_into(mask, w, h, u, b, r);
  double s = det_dot(r, r, n);
  free(r);
  return s;
}

/* ---- partition: partition.hpp:46-106 ----------------------------------- */
void or_partition_axis(int extent, int block, int overlap, int* anchors, int* count,
                       int* owned_end) {
  int stride = block - overlap;
  int n = 1;
  if (extent > block) n = (extent - block + stride - 1) / stride + 1;
  for (int k = 0; k + 1 < n; ++k) anchors[k] = k * stride;
  anchors[n - 1] = extent - block;
  for (int k = 0; k < n; ++k) {
    owned_end[k] = (k + 1 == n) ? extent : (anchors[k] + anchors[k + 1] + block - 1) / 2 + 1;
  }
  *count = n;
}

/* ---- local block structure: schwarz.hpp:84-111, 179-198 ---------------- */
typedef struct {
  int bw, bh, wp;    /* block extent, padded row stride */
  size_t padded;
  double *unk, *knw, *diag, *pv, *rhs, *x, *r, *p, *Ap;
} local_scratch;

static void scratch_init(local_scratch* s, int bw, int bh) {
  s->bw = bw;
  s->bh = bh;
  s->wp = bw + 2;
  s->padded = (size_t)(bw + 2) * (bh + 2);
  double* mem = (double*)calloc(9 * s->padded, sizeof(double));
  s->unk = mem;
  s->knw = mem + s->padded;
  s->diag = mem + 2 * s->padded;
  s->pv = mem + 3 * s->padded;
  s->rhs = mem + 4 * s->padded;
  s->x = mem + 5 * s->padded;
  s->r = mem + 6 * s->padded;
  s->p = mem + 7 * s->padded;
  s->Ap = mem + 8 * s->padded;
}

static void scratch_free(local_scratch* s) { free(s->unk); }

/* fill_local_structure + prepare_local_block; returns the unknown count. */
static size_t prepare_block(const uint8_t* mask, int w, int h, int x0, int y0,
                            int flavour, double alpha, local_scratch* s) {
  memset(s->unk, 0, 3 * s->padded * sizeof(double));  /* unk, knw, diag */
  size_t m = 0;
  for (int ly = 0; ly < s->bh; ++ly) {
    int gy = y0 + ly;
    for (int lx = 0; lx < s->bw; ++lx) {
      int gx = x0 + lx;
      size_t cell = (size_t)(ly + 1) * s->wp + lx + 1;
      int known = mask[(size_t)gy * w + gx] != 0;
      s->knw[cell] = known;
      if (known) {
        s->diag[cell] = 1.0;
      } else {
        int deg = (gx > 0) + (gx + 1 < w) + (gy > 0) + (gy + 1 < h);
        int cut = (gx > 0 && lx == 0) + (gx + 1 < w && lx + 1 == s->bw) + (gy > 0 && ly == 0) +
                  (gy + 1 < h && ly + 1 == s->bh);
        s->diag[cell] = flavour == 0 ? (double)deg : deg + (alpha - 1.0) * cut;
      }
      s->unk[cell] = 1.0 - s->knw[cell];
      m += s->knw[cell] == 0.0;
    }
  }
  return m;
}

/* LocalStencilOperator::apply (schwarz.hpp:146-159). */
static void local_apply(const local_scratch* s, const double* v, double* out) {
  int wp = s->wp;
  for (int row = 1; row <= s->bh; ++row) {
    size_t off = (size_t)row * wp;
    const double* vc = v + off;
    const double* d = s->diag + off;
    const double* u = s->unk + off;
    double* o = out + off;
    for (int col = 1; col <= s->bw; ++col) {
      o[col] = u[col] * (d[col] * vc[col] - vc[col - 1] - vc[col + 1] - vc[col - wp] -
                         vc[col + wp]);
    }
  }
}

/* cg_solve (cg.hpp:90-154) from x = 0 on the padded local system.
 * Returns 1 when converged; *iters receives report.iterations. */
static int local_cg(local_scratch* s, double tol, int max_it, int check, int* iters) {
  size_t n = s->padded;
  double *x = s->x, *r = s->r, *p = s->p, *Ap = s->Ap, *b = s->rhs;
  *iters = 0;
  memset(x, 0, n * sizeof(double));
  memset(r, 0, n * sizeof(double));
  memset(Ap, 0, n * sizeof(double));
  local_apply(s, x, r);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double r0 = det_norm(r, n);
  if (r0 == 0.0) return 1;
  memcpy(p, r, n * sizeof(double));
  double rr = det_dot(r, r, n);
  for (int iter = 1; iter <= max_it; ++iter) {
    local_apply(s, p, Ap);
    double pAp = det_dot(p, Ap, n);
    if (!(pAp > 0.0) || !isfinite(pAp)) {  /* breakdown guard cg.hpp:120-125 */
      *iters = iter - 1;
      return 0;
    }
    double a = rr / pAp;
    for (size_t i = 0; i < n; ++i) x[i] += a * p[i];
    for (size_t i = 0; i < n; ++i) r[i] += -a * Ap[i];
    double rr_new = det_dot(r, r, n);
    int cadence = iter % check == 0 || iter == max_it;
    int maybe_done = sqrt(rr_new) <= tol * r0;
    if (cadence || maybe_done) {  /* true residual, cg.hpp:131-146 */
      local_apply(s, x, Ap);
      for (size_t i = 0; i < n; ++i) Ap[i] = b[i] - Ap[i];
      double rel = det_norm(Ap, n) / r0;
      if (rel <= tol) {
        *iters = iter;
        return 1;
      }
      memcpy(r, Ap, n * sizeof(double));
      rr_new = det_dot(r, r, n);
    }
    double beta = rr_new / rr;
    for (size_t i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    rr = rr_new;
  }
  *iters = max_it;
  return 0;
}

/* solve_local_block (schwarz.hpp:202-250): v (cell-ordered residual slice)
 * is overwritten with the local correction. */
static int solve_block(local_scratch* s, size_t m, const or_options* opt, double* v,
                       long long* cg_iters) {
  if (m == 0) return 1;
  int wp = s->wp;
  memset(s->pv, 0, s->padded * sizeof(double));
  for (int ly = 0; ly < s->bh; ++ly) {
    memcpy(s->pv + (size_t)(ly + 1) * wp + 1, v + (size_t)ly * s->bw, s->bw * sizeof(double));
  }
  memset(s->rhs, 0, s->padded * sizeof(double));
  for (int row = 1; row <= s->bh; ++row) {
    size_t off = (size_t)row * wp;
    const double* pv = s->pv + off;
    const double* kn = s->knw + off;
    const double* u = s->unk + off;
    double* rhs = s->rhs + off;
    for (int col = 1; col <= s->bw; ++col) {
      rhs[col] = u[col] * (pv[col] + kn[col - 1] * pv[col - 1] + kn[col + 1] * pv[col + 1] +
                           kn[col - wp] * pv[col - wp] + kn[col + wp] * pv[col + wp]);
    }
  }
  int iters = 0;
  int ok = local_cg(s, opt->local_tolerance, opt->local_max_iterations, opt->local_check_interval,
                    &iters);
  *cg_iters += iters;
  for (int ly = 0; ly < s->bh; ++ly) {
    size_t off = (size_t)(ly + 1) * wp + 1;
    for (int lx = 0; lx < s->bw; ++lx) {
      if (s->unk[off + lx] != 0.0) v[(size_t)ly * s->bw + lx] = s->x[off + lx];
    }
  }
  return ok;
}

/* One sweep of the block loop in run_schwarz_level (schwarz.hpp:305-318),
 * with the residual r = b - A u precomputed per channel. */
static void sweep_with_residual(const uint8_t* mask, int w, int h, int c, const double* r,
                                double* u, int block, int overlap, const or_options* opt,
                                long long* failures, long long* cg_iters) {
  int nx, ny;
  int* ax = (int*)malloc(sizeof(int) * 4 * (size_t)(w + h + 2));
  int* ex = ax + (w + h + 2);
  int* ay = ex + (w + h + 2);
  int* ey = ay + (w + h + 2);
  or_partition_axis(w, block, overlap, ax, &nx, ex);
  or_partition_axis(h, block, overlap, ay, &ny, ey);
  size_t n = (size_t)w * h;
  local_scratch s;
  scratch_init(&s, block, block);
  double* v = (double*)malloc((size_t)block * block * sizeof(double));
  for (int by = 0; by < ny; ++by) {
    for (int bx = 0; bx < nx; ++bx) {
      int x0 = ax[bx], y0 = ay[by];
      int ox0 = bx == 0 ? 0 : ex[bx - 1], ox1 = ex[bx];
      int oy0 = by == 0 ? 0 : ey[by - 1], oy1 = ey[by];
      size_t m = prepare_block(mask, w, h, x0, y0, opt->flavour, opt->alpha, &s);
      for (int ch = 0; ch < c; ++ch) {
        const double* rc = r + (size_t)ch * n;
        double* uc = u + (size_t)ch * n;
        for (int ly = 0; ly < block; ++ly)  /* restrict_block_into, partition.hpp:109-121 */
          memcpy(v + (size_t)ly * block, rc + (size_t)(y0 + ly) * w + x0, block * sizeof(double));
        if (!solve_block(&s, m, opt, v, cg_iters)) ++*failures;
        for (int y = oy0; y < oy1; ++y)  /* accumulate_owned, partition.hpp:148-156 */
          for (int x = ox0; x < ox1; ++x)
            uc[(size_t)y * w + x] += v[(size_t)(y - y0) * block + (x - x0)];
      }
    }
  }
  free(v);
  free(ax);
  scratch_free(&s);
}

void or_schwarz_sweep(const uint8_t* mask, int w, int h, int c, const double* b, const double* u,
                      int block, int overlap, const or_options* opt, double* u_new,
                      long long* failures, long long* cg_iterations) {
  size_t n = (size_t)w * h;
  double* r = (double*)malloc((size_t)c * n * sizeof(double));
  for (int ch = 0; ch < c; ++ch) residual_into(mask, w, h, u + ch * n, b + ch * n, r + ch * n);
  memcpy(u_new, u, (size_t)c * n * sizeof(double));
  sweep_with_residual(mask, w, h, c, r, u_new, block, overlap, opt, failures, cg_iterations);
  free(r);
}

void or_local_operator_apply(const uint8_t* mask, int w, int h, int x0, int y0, int bw, int bh,
                             int flavour, double alpha, const double* v, double* out) {
  /* LocalOperator::apply (schwarz.hpp:57-75) over build_local_operator's
   * structure (schwarz.hpp:115-130). */
  for (int ly = 0; ly < bh; ++ly) {
    for (int lx = 0; lx < bw; ++lx) {
      int gx = x0 + lx, gy = y0 + ly;
      size_t i = (size_t)ly * bw + lx;
      if (mask[(size_t)gy * w + gx]) {
        out[i] = v[i];
        continue;
      }
      int deg = (gx > 0) + (gx + 1 < w) + (gy > 0) + (gy + 1 < h);
      int cut = (gx > 0 && lx == 0) + (gx + 1 < w && lx + 1 == bw) + (gy > 0 && ly == 0) +
                (gy + 1 < h && ly + 1 == bh);
      double d = flavour == 0 ? (double)deg : deg + (alpha - 1.0) * cut;
      double acc = d * v[i];
      if (lx > 0) acc -= v[i - 1];
      if (lx + 1 < bw) acc -= v[i + 1];
      if (ly > 0) acc -= v[i - bw];
      if (ly + 1 < bh) acc -= v[i + bw];
      out[i] = acc;
    }
  }
}

/* ---- run_schwarz_level: schwarz.hpp:266-323 --------------------------- */
static int axis_count(int extent, int block, int overlap) {
  int stride = block - overlap;
  return extent > block ? (extent - block + stride - 1) / stride + 1 : 1;
}

typedef struct {
  int iterations;
  double final_rel;
  int converged;
} level_outcome;

static level_outcome run_level(const uint8_t* mask, int w, int h, int c, const double* b,
                               double* u, double r0, double tol, int block, int overlap,
                               const or_options* opt, or_report* rep, double* trace,
                               int trace_cap, int sink) {
  size_t n = (size_t)w * h;
  double* r = (double*)malloc((size_t)c * n * sizeof(double));
  level_outcome out = {0, 0.0, 0};
  for (int outer = 0;; ++outer) {
    double joint_sq = 0.0;
    for (int ch = 0; ch < c; ++ch) {
      residual_into(mask, w, h, u + ch * n, b + ch * n, r + ch * n);
      double nrm = det_norm(r + ch * n, n);
      joint_sq = fma(nrm, nrm, joint_sq);  /* contracted in the reference build */
    }
    double rel = r0 > 0.0 ? sqrt(joint_sq) / r0 : 0.0;
    if (sink) {
      if (rep->trace_rows < trace_cap && trace) trace[rep->trace_rows] = rel;
      rep->trace_rows++;
    }
    out.iterations = outer;
    out.final_rel = rel;
    if (rel <= tol) {
      out.converged = 1;
      break;
    }
    if (outer >= opt->max_outer_iterations) break;
    sweep_with_residual(mask, w, h, c, r, u, block, overlap, opt, &rep->local_failures,
                        &rep->local_cg_iterations);
    rep->local_solves += (long long)axis_count(w, block, overlap) * axis_count(h, block, overlap) * c;
  }
  free(r);
  return out;
}

/* canonical_r0 (schwarz.hpp:333-345, cg.hpp:172-185). */
static double canonical_r0(const uint8_t* mask, int w, int h, int c, const double* b,
                           int normalizer) {
  size_t n = (size_t)w * h;
  double acc = 0.0;
  if (normalizer == 1) {
    for (int ch = 0; ch < c; ++ch) {
      double nrm = det_norm(b + ch * n, n);
      acc = fma(nrm, nrm, acc);
    }
    return sqrt(acc);
  }
  double* r = (double*)malloc(n * sizeof(double));
  for (int ch = 0; ch < c; ++ch) {
    residual_into(mask, w, h, b + ch * n, b + ch * n, r);
    double nrm = det_norm(r, n);
    acc += nrm * nrm;
  }
  free(r);
  return sqrt(acc);
}

/* ---- CG level solver: reduction.hpp:26-145, cg.hpp:192-291,
 *      multilevel.hpp:162-209 ---------------------------------------------- */
typedef struct {
  int w, h;
  size_t n;            /* reduced size */
  int32_t* unknown_of; /* pixel -> reduced index or -1 */
  int32_t* pixel_of;
  double* diag;
} reduced_sys;

static reduced_sys reduce_structure(const uint8_t* mask, int w, int h) {
  reduced_sys s;
  s.w = w;
  s.h = h;
  size_t np = (size_t)w * h;
  s.unknown_of = (int32_t*)malloc(np * sizeof(int32_t));
  s.pixel_of = (int32_t*)malloc(np * sizeof(int32_t));
  s.n = 0;
  for (size_t i = 0; i < np; ++i) {
    s.unknown_of[i] = -1;
    if (!mask[i]) {
      s.unknown_of[i] = (int32_t)s.n;
      s.pixel_of[s.n++] = (int32_t)i;
    }
  }
  s.diag = (double*)malloc((s.n + 1) * sizeof(double));
  for (size_t k = 0; k < s.n; ++k) {
    int p = s.pixel_of[k], x = p % w, y = p / w;
    s.diag[k] = (x > 0) + (x + 1 < w) + (y > 0) + (y + 1 < h);
  }
  return s;
}

static void reduced_free(reduced_sys* s) {
  free(s->unknown_of);
  free(s->pixel_of);
  free(s->diag);
}

/* ReducedSystem::apply (reduction.hpp:36-58) */
static void reduced_apply(const reduced_sys* s, const double* x, double* y) {
  int w = s->w;
  for (size_t k = 0; k < s->n; ++k) {
    int32_t p = s->pixel_of[k];
    int x_ = p % w, y_ = p / w;
    double acc = s->diag[k] * x[k];
    if (x_ > 0 && s->unknown_of[p - 1] >= 0) acc -= x[s->unknown_of[p - 1]];
    if (x_ + 1 < w && s->unknown_of[p + 1] >= 0) acc -= x[s->unknown_of[p + 1]];
    if (y_ > 0 && s->unknown_of[p - w] >= 0) acc -= x[s->unknown_of[p - w]];
    if (y_ + 1 < s->h && s->unknown_of[p + w] >= 0) acc -= x[s->unknown_of[p + w]];
    y[k] = acc;
  }
}

/* cg_solve_lockstep (cg.hpp:192-291); sets *iters / *final_rel, returns converged. */
static int cg_lockstep(const reduced_sys* s, double** b, double** x, int nc, double tol, int maxit,
                       int check, double external_r0, double** u_obs, const double* bfull,
                       size_t npix, or_report* rep, double* trace, int trace_cap, int sink,
                       int* iters, double* final_rel) {
  size_t n = s->n;
  *iters = 0;
  if (n == 0) {
    *final_rel = 0.0;
    return 1;
  }
  double** r = (double**)malloc(nc * sizeof(double*));
  double** p = (double**)malloc(nc * sizeof(double*));
  double* Ap = (double*)malloc(n * sizeof(double));
  double *rr = (double*)calloc(nc, sizeof(double)), *rr_next = (double*)calloc(nc, sizeof(double));
  char* frozen = (char*)calloc(nc, 1);
  double joint0_sq = 0.0;
  for (int c = 0; c < nc; ++c) {
    r[c] = (double*)malloc(n * sizeof(double));
    p[c] = (double*)malloc(n * sizeof(double));
    reduced_apply(s, x[c], r[c]);
    for (size_t i = 0; i < n; ++i) r[c][i] = b[c][i] - r[c][i];
    rr[c] = det_dot(r[c], r[c], n);
    joint0_sq += rr[c];
    memcpy(p[c], r[c], n * sizeof(double));
  }
  double r0 = external_r0 > 0.0 ? external_r0 : sqrt(joint0_sq);
  int converged = 0, done = 0;
  if (r0 == 0.0 || sqrt(joint0_sq) <= tol * r0) {
    *final_rel = r0 == 0.0 ? 0.0 : sqrt(joint0_sq) / r0;
    converged = done = 1;
  }
  double freeze_sq = 1e-4 * tol * tol * r0 * r0;
  double rel = done ? *final_rel : sqrt(joint0_sq) / r0;
  for (int iter = 1; !done && iter <= maxit; ++iter) {
    double joint_sq = 0.0;
    int broke = 0;
    for (int c = 0; c < nc; ++c) {
      if (frozen[c] || rr[c] <= freeze_sq) {
        frozen[c] = 1;
        rr_next[c] = rr[c];
        joint_sq += rr[c];
        continue;
      }
      reduced_apply(s, p[c], Ap);
      double pAp = det_dot(p[c], Ap, n);
      if (!(pAp > 0.0) || !isfinite(pAp)) {
        *iters = iter - 1;
        *final_rel = rel;
        broke = 1;
        break;
      }
      double alpha = rr[c] / pAp;
      for (size_t i = 0; i < n; ++i) x[c][i] += alpha * p[c][i];
      for (size_t i = 0; i < n; ++i) r[c][i] += -alpha * Ap[i];
      rr_next[c] = det_dot(r[c], r[c], n);
      joint_sq += rr_next[c];
    }
    if (broke) {
      done = 1;
      break;
    }
    int cadence = iter % check == 0 || iter == maxit;
    int maybe_done = sqrt(joint_sq) <= tol * r0;
    if (cadence || maybe_done) {
      double true_sq = 0.0;
      for (int c = 0; c < nc; ++c) {
        reduced_apply(s, x[c], Ap);
        for (size_t i = 0; i < n; ++i) Ap[i] = b[c][i] - Ap[i];
        double nc2 = det_dot(Ap, Ap, n);
        true_sq += nc2;
        if (!frozen[c]) {
          memcpy(r[c], Ap, n * sizeof(double));
          rr_next[c] = nc2;
        }
      }
      rel = sqrt(true_sq) / r0;
      if (sink) {
        if (trace && rep->trace_rows < trace_cap) trace[rep->trace_rows] = rel;
        rep->trace_rows++;
      }
      if (rel <= tol) {
        *iters = iter;
        *final_rel = rel;
        converged = done = 1;
        break;
      }
    }
    for (int c = 0; c < nc; ++c) {
      if (frozen[c]) continue;
      double beta = rr[c] > 0.0 ? rr_next[c] / rr[c] : 0.0;
      for (size_t i = 0; i < n; ++i) p[c][i] = r[c][i] + beta * p[c][i];
      rr[c] = rr_next[c];
    }
    if (iter == maxit) {
      *iters = maxit;
      *final_rel = rel;
    }
  }
  if (!done && maxit <= 0) {
    *iters = maxit < 0 ? 0 : maxit;
    *final_rel = rel;
  }
  (void)u_obs;
  (void)bfull;
  (void)npix;
  for (int c = 0; c < nc; ++c) {
    free(r[c]);
    free(p[c]);
  }
  free(r);
  free(p);
  free(Ap);
  free(rr);
  free(rr_next);
  free(frozen);
  return converged;
}

/* run_cg_level (multilevel.hpp:162-209) */
static level_outcome run_cg_level(const uint8_t* mask, int w, int h, int c, const double* bvals,
                                  double* u, double tol, const or_options* opt, or_report* rep,
                                  double* trace, int trace_cap, int sink) {
  size_t np = (size_t)w * h;
  reduced_sys s = reduce_structure(mask, w, h);
  size_t n = s.n;
  double** rhs = (double**)malloc(c * sizeof(double*));
  double** x = (double**)malloc(c * sizeof(double*));
  double* tmp = (double*)malloc((n + 1) * sizeof(double));
  double r0_sq = 0.0, init_sq = 0.0;
  for (int k = 0; k < c; ++k) {
    const double* b = bvals + k * np;  /* build_rhs(values) == values */
    rhs[k] = (double*)malloc((n + 1) * sizeof(double));
    for (size_t q = 0; q < n; ++q) {  /* reduced_rhs (reduction.hpp:119-134) */
      int32_t p = s.pixel_of[q];
      int xx = p % w, yy = p / w;
      double acc = b[p];
      if (xx > 0 && s.unknown_of[p - 1] == -1) acc += b[p - 1];
      if (xx + 1 < w && s.unknown_of[p + 1] == -1) acc += b[p + 1];
      if (yy > 0 && s.unknown_of[p - w] == -1) acc += b[p - w];
      if (yy + 1 < h && s.unknown_of[p + w] == -1) acc += b[p + w];
      rhs[k][q] = acc;
    }
    double nrm = det_norm(rhs[k], n);
    r0_sq = fma(nrm, nrm, r0_sq);
    x[k] = (double*)malloc((n + 1) * sizeof(double));
    for (size_t q = 0; q < n; ++q) x[k][q] = u[k * np + s.pixel_of[q]];
  }
  double r0 = sqrt(r0_sq);
  for (int k = 0; k < c; ++k) {
    reduced_apply(&s, x[k], tmp);
    for (size_t q = 0; q < n; ++q) tmp[q] = rhs[k][q] - tmp[q];
    double nrm = det_norm(tmp, n);
    init_sq = fma(nrm, nrm, init_sq);
  }
  double rel0 = r0 > 0.0 ? sqrt(init_sq) / r0 : 0.0;
  if (sink) {
    if (trace && rep->trace_rows < trace_cap) trace[rep->trace_rows] = rel0;
    rep->trace_rows++;
  }
  level_outcome out = {0, 0.0, 0};
  out.converged = cg_lockstep(&s, rhs, x, c, tol, opt->cg_max_iterations, opt->cg_check_interval,
                              r0, NULL, NULL, np, rep, trace, trace_cap, sink, &out.iterations,
                              &out.final_rel);
  for (int k = 0; k < c; ++k) {  /* embed_solution (reduction.hpp:138-145) */
    const double* b = bvals + k * np;
    for (size_t i = 0; i < np; ++i) u[k * np + i] = b[i];
    for (size_t q = 0; q < n; ++q) u[k * np + s.pixel_of[q]] = x[k][q];
    free(rhs[k]);
    free(x[k]);
  }
  free(rhs);
  free(x);
  free(tmp);
  reduced_free(&s);
  return out;
}

/* ---- pyramid: multilevel.hpp:33-128 ------------------------------------ */
int or_restrict_level(const uint8_t* mask, const double* values, int fw, int fh, int c,
                      int averaging, uint8_t* cmask, double* cvalues) {
  if (fw < 2 || fh < 2) return 1;
  int cw = (fw + 1) / 2, ch = (fh + 1) / 2;
  size_t fn = (size_t)fw * fh, cn = (size_t)cw * ch;
  memset(cmask, 0, cn);
  memset(cvalues, 0, (size_t)c * cn * sizeof(double));
  for (int cy = 0; cy < ch; ++cy) {
    int fy0 = 2 * cy, fy1 = fy0 + 2 < fh ? fy0 + 2 : fh;
    for (int cx = 0; cx < cw; ++cx) {
      int fx0 = 2 * cx, fx1 = fx0 + 2 < fw ? fx0 + 2 : fw;
      int known = 0, total = 0;
      for (int y = fy0; y < fy1; ++y)
        for (int x = fx0; x < fx1; ++x) {
          known += mask[(size_t)y * fw + x] != 0;
          ++total;
        }
      if (known == 0) continue;
      cmask[(size_t)cy * cw + cx] = 1;
      for (int k = 0; k < c; ++k) {
        double acc = 0.0;
        for (int y = fy0; y < fy1; ++y)
          for (int x = fx0; x < fx1; ++x) {
            if (averaging == 0 && !mask[(size_t)y * fw + x]) continue;
            acc += values[k * fn + (size_t)y * fw + x];
          }
        cvalues[k * cn + (size_t)cy * cw + cx] = acc / (averaging == 0 ? known : total);
      }
    }
  }
  return 0;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

void or_prolongate(const double* coarse, int cw, int ch, int fw, int fh, double* fine) {
  for (int fy = 0; fy < fh; ++fy) {
    double yc = clampd(0.5 * fy - 0.25, 0.0, (double)(ch - 1));
    int y0 = (int)yc;
    int y1 = y0 + 1 < ch - 1 ? y0 + 1 : ch - 1;
    double ty = yc - y0;
    for (int fx = 0; fx < fw; ++fx) {
      double xc = clampd(0.5 * fx - 0.25, 0.0, (double)(cw - 1));
      int x0 = (int)xc;
      int x1 = x0 + 1 < cw - 1 ? x0 + 1 : cw - 1;
      double tx = xc - x0;
      double v00 = coarse[(size_t)y0 * cw + x0];
      double v01 = coarse[(size_t)y0 * cw + x1];
      double v10 = coarse[(size_t)y1 * cw + x0];
      double v11 = coarse[(size_t)y1 * cw + x1];
      fine[(size_t)fy * fw + fx] =
          (1.0 - ty) * ((1.0 - tx) * v00 + tx * v01) + ty * ((1.0 - tx) * v10 + tx * v11);
    }
  }
}

/* ---- multilevel_solve: multilevel.hpp:239-310 -------------------------- */
int or_multilevel_solve(const double* f, const uint8_t* mask, int w, int h, int c,
                        const or_options* opt, double* out, or_report* rep, double* trace_rel,
                        int trace_cap) {
  memset(rep, 0, sizeof(*rep));
  if (w <= 0 || h <= 0 || c <= 0 || opt->levels < 1 || !(opt->tolerance > 0.0) ||
      !(opt->coarse_tolerance > 0.0)) {
    rep->error = 1;
    return 1;
  }
  size_t kn = 0;
  for (size_t i = 0; i < (size_t)w * h; ++i) kn += mask[i] != 0;
  if (kn == 0) {  /* build_rhs rejects an empty mask, operators.hpp:83 */
    rep->error = 1;
    return 1;
  }
  /* build_pyramid (multilevel.hpp:74-96) */
  int lw[OR_MAX_LEVELS], lh[OR_MAX_LEVELS];
  uint8_t* lm[OR_MAX_LEVELS];
  double* lv[OR_MAX_LEVELS];
  int depth = 1;
  lw[0] = w;
  lh[0] = h;
  size_t n0 = (size_t)w * h;
  lm[0] = (uint8_t*)malloc(n0);
  memcpy(lm[0], mask, n0);
  lv[0] = (double*)malloc((size_t)c * n0 * sizeof(double));
  for (int k = 0; k < c; ++k)
    for (size_t i = 0; i < n0; ++i) lv[0][k * n0 + i] = mask[i] ? f[k * n0 + i] : 0.0;
  while (depth < opt->levels && depth < OR_MAX_LEVELS) {
    int fw = lw[depth - 1], fh = lh[depth - 1];
    if (fw < 2 || fh < 2) break;
    int cw = (fw + 1) / 2, chh = (fh + 1) / 2;
    lw[depth] = cw;
    lh[depth] = chh;
    lm[depth] = (uint8_t*)malloc((size_t)cw * chh);
    lv[depth] = (double*)malloc((size_t)c * cw * chh * sizeof(double));
    or_restrict_level(lm[depth - 1], lv[depth - 1], fw, fh, c, opt->averaging, lm[depth],
                      lv[depth]);
    ++depth;
  }
  rep->depth = depth;

  double* u = NULL;
  int coarse_capped = 0;
  for (int level = depth - 1; level >= 0; --level) {
    int W = lw[level], H = lh[level];
    size_t n = (size_t)W * H;
    /* b = build_rhs(values) equals values: unknowns are already zero. */
    const double* b = lv[level];
    if (level == depth - 1) {
      u = (double*)malloc((size_t)c * n * sizeof(double));
      memcpy(u, b, (size_t)c * n * sizeof(double));
    }
    int finest = level == 0;
    double tol = finest ? opt->tolerance : opt->coarse_tolerance;
    /* clamped_partition (multilevel.hpp:146-150) */
    int be = opt->block_size < W ? opt->block_size : W;
    be = be < H ? be : H;
    int oe = opt->overlap < be - 1 ? opt->overlap : be - 1;
    if (oe < 0) oe = 0;
    level_outcome o;
    if (opt->flavour == 2) {
      o = run_cg_level(lm[level], W, H, c, b, u, tol, opt, rep, trace_rel, trace_cap, finest);
    } else {
      double r0 = canonical_r0(lm[level], W, H, c, b, opt->normalizer);
      o = run_level(lm[level], W, H, c, b, u, r0, tol, be, oe, opt, rep, trace_rel, trace_cap,
                    finest);
    }
    rep->level_iterations[level] = o.iterations;
    rep->level_final_rel[level] = o.final_rel;
    rep->level_converged[level] = o.converged;
    if (finest) {
      rep->iterations = o.iterations;
      rep->final_rel = o.final_rel;
      rep->converged = o.converged;
    } else {
      if (!o.converged) coarse_capped = 1;
      int fw = lw[level - 1], fh = lh[level - 1];
      size_t fn = (size_t)fw * fh;
      double* un = (double*)malloc((size_t)c * fn * sizeof(double));
      for (int k = 0; k < c; ++k) {
        or_prolongate(u + k * n, W, H, fw, fh, un + k * fn);
        for (size_t i = 0; i < fn; ++i)
          if (lm[level - 1][i]) un[k * fn + i] = lv[level - 1][k * fn + i];
      }
      free(u);
      u = un;
    }
  }
  (void)coarse_capped;
  memcpy(out, u, (size_t)c * n0 * sizeof(double));
  free(u);
  for (int l = 0; l < depth; ++l) {
    free(lm[l]);
    free(lv[l]);
  }
  return 0;
}

/* ---- Voronoi densification: masks.hpp:45-215 ---------------------------- */

/* Exact nearest known pixel under squared Euclidean distance, ties to the
 * lower site index (assign_nearest_site, masks.hpp:54-139).  Same search as
 * the reference: sites are binned on a square grid of side
 * max(1, floor(sqrt(n/m))) and rings of bins are visited around the pixel's
 * bin until the ring's minimum possible distance exceeds the best one found;
 * bins whose rectangle is farther than the best are skipped.  The result is
 * the lexicographic minimum of (distance, site index) over all sites. */
int or_assign_nearest_site(const uint8_t* mask, int w, int h, int32_t* sites, int32_t* site_of,
                           int* num_sites) {
  const size_t n = (size_t)w * h;
  int m = 0;
  for (size_t i = 0; i < n; ++i)
    if (mask[i]) sites[m++] = (int32_t)i;
  *num_sites = m;
  if (m == 0) return 1;
  int cell = (int)sqrt((double)n / m);
  if (cell < 1) cell = 1;
  const int gw = (w + cell - 1) / cell, gh = (h + cell - 1) / cell;
  const size_t nb = (size_t)gw * gh;
  int32_t* start = (int32_t*)calloc(nb + 1, sizeof(int32_t));
  int32_t* members = (int32_t*)malloc((size_t)m * sizeof(int32_t));
  int32_t* fill = (int32_t*)malloc(nb * sizeof(int32_t));
  for (int s = 0; s < m; ++s) {
    int x = sites[s] % w, y = sites[s] / w;
    start[(size_t)(y / cell) * gw + x / cell + 1]++;
  }
  for (size_t b = 0; b < nb; ++b) start[b + 1] += start[b];
  memcpy(fill, start, nb * sizeof(int32_t));
  for (int s = 0; s < m; ++s) {
    int x = sites[s] % w, y = sites[s] / w;
    members[fill[(size_t)(y / cell) * gw + x / cell]++] = s;
  }
  const int rings = gw > gh ? gw : gh;
  for (int py = 0; py < h; ++py) {
    for (int px = 0; px < w; ++px) {
      const int cx = px / cell, cy = py / cell;
      long long best_d = -1;
      int best = -1;
      for (int ring = 0; ring <= rings; ++ring) {
        if (best >= 0 && ring >= 1) {
          long long reach = (long long)(ring - 1) * cell + 1;
          if (reach * reach > best_d) break;
        }
        for (int by = cy - ring; by <= cy + ring; ++by) {
          if (by < 0 || by >= gh) continue;
          int edge_row = by == cy - ring || by == cy + ring;
          int step = edge_row ? 1 : 2 * ring;
          for (int bx = cx - ring; bx <= cx + ring; bx += step > 0 ? step : 1) {
            if (bx < 0 || bx >= gw) continue;
            int x0 = bx * cell, x1 = x0 + cell - 1, y0 = by * cell, y1 = y0 + cell - 1;
            if (x1 > w - 1) x1 = w - 1;
            if (y1 > h - 1) y1 = h - 1;
            long long dx = px < x0 ? x0 - px : (px > x1 ? px - x1 : 0);
            long long dy = py < y0 ? y0 - py : (py > y1 ? py - y1 : 0);
            if (best >= 0 && dx * dx + dy * dy > best_d) continue;
            size_t b = (size_t)by * gw + bx;
            for (int k = start[b]; k < start[b + 1]; ++k) {
              int s = members[k];
              long long ex = sites[s] % w - px, ey = sites[s] / w - py;
              long long d = ex * ex + ey * ey;
              if (best < 0 || d < best_d || (d == best_d && s < best)) {
                best_d = d;
                best = s;
              }
            }
            if (step == 0) break;
          }
        }
      }
      site_of[(size_t)py * w + px] = best;
    }
  }
  free(start);
  free(members);
  free(fill);
  return 0;
}

typedef struct {
  double err;
  long long area;
  int index;
} cell_rank;

/* Ranking of masks.hpp:189-194: error desc, area desc, site index asc. */
static int cell_rank_cmp(const void* pa, const void* pb) {
  const cell_rank* a = (const cell_rank*)pa;
  const cell_rank* b = (const cell_rank*)pb;
  if (a->err != b->err) return a->err > b->err ? -1 : 1;
  if (a->area != b->area) return a->area > b->area ? -1 : 1;
  return a->index < b->index ? -1 : (a->index > b->index);
}

/* voronoi_densify (masks.hpp:155-212) from a given seed mask (the caller
 * draws it with random_mask, masks.hpp:170).  Each sweep: inpaint with the
 * multilevel ORAS solver at inner_tolerance, assign Voronoi cells, sum the
 * squared error of the unknown pixels of every cell in pixel order, rank the
 * cells and plant a known pixel at the worst pixel of the first
 * max(1, floor(cell_fraction * m)) cells (capped by the cells with pixels and
 * by the remaining target). */
int or_voronoi_densify(const double* f, int w, int h, int c, const uint8_t* seed_mask,
                       long long target_k, double cell_fraction, double inner_tolerance,
                       int max_sweeps, const or_options* solve, uint8_t* mask, int* sweeps) {
  const size_t n = (size_t)w * h;
  memcpy(mask, seed_mask, n);
  long long known = 0;
  for (size_t i = 0; i < n; ++i) known += mask[i] != 0;
  or_options so = *solve;
  so.tolerance = inner_tolerance;
  so.flavour = 1;
  double* u = (double*)malloc((size_t)c * n * sizeof(double));
  int32_t* sites = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* site_of = (int32_t*)malloc(n * sizeof(int32_t));
  cell_rank* cells = (cell_rank*)malloc(n * sizeof(cell_rank));
  double* worst_e = (double*)malloc(n * sizeof(double));
  int32_t* worst_p = (int32_t*)malloc(n * sizeof(int32_t));
  int rc = 0;
  *sweeps = 0;
  while (known < target_k && *sweeps < max_sweeps) {
    or_report rep;
    if (or_multilevel_solve(f, mask, w, h, c, &so, u, &rep, NULL, 0)) {
      rc = 1;
      break;
    }
    int m = 0;
    or_assign_nearest_site(mask, w, h, sites, site_of, &m);
    for (int s = 0; s < m; ++s) {
      cells[s].err = 0.0;
      cells[s].area = 0;
      cells[s].index = s;
      worst_e[s] = -1.0;
      worst_p[s] = -1;
    }
    for (size_t p = 0; p < n; ++p) {
      if (mask[p]) continue;
      int s = site_of[p];
      double e = 0.0;
      for (int k = 0; k < c; ++k) {
        double d = u[k * n + p] - f[k * n + p];
        e = fma(d, d, e);
      }
      cells[s].err += e;
      cells[s].area++;
      if (e > worst_e[s]) {
        worst_e[s] = e;
        worst_p[s] = (int32_t)p;
      }
    }
    int used = 0;
    for (int s = 0; s < m; ++s)
      if (cells[s].area > 0) cells[used++] = cells[s];
    qsort(cells, (size_t)used, sizeof(cell_rank), cell_rank_cmp);
    long long quota = (long long)(cell_fraction * (double)m);
    if (quota < 1) quota = 1;
    if (quota > used) quota = used;
    if (quota > target_k - known) quota = target_k - known;
    for (long long i = 0; i < quota; ++i) mask[worst_p[cells[i].index]] = 1;
    known += quota;
    ++*sweeps;
  }
  free(u);
  free(sites);
  free(site_of);
  free(cells);
  free(worst_e);
  free(worst_p);
  return rc;
}
