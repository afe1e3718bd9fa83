"""CPU: the C ABI library loads, exports every declared symbol, and its
host-only logic (partition, generators, option validation) matches the
reference.  No device computation here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2110_03946_b200 as si
from paper_2110_03946_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "schwarz_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(si_[a-z0-9_]+)\s*\(", text)) - {"si_trace_fn"})


def test_library_exports_every_declared_symbol():
    lib = L.load()
    names = declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
        assert n in L.SIGNATURES, f"{n} not bound in _lib.SIGNATURES"
    assert set(L.SIGNATURES) == set(names)


def test_library_is_sm100a_cuda():
    out = subprocess.run(["cuobjdump", "--list-elf", L.lib_path()], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_default_options_are_reference_defaults():
    o = L.si_options()
    L.load().si_default_options(C.byref(o))
    assert (o.tolerance, o.levels, o.block_size, o.overlap, o.alpha, o.coarse_tolerance) == \
        (1e-3, 3, 32, 6, 0.25, 1e-2)
    assert (o.local_tolerance, o.local_max_iterations, o.local_check_interval) == (1e-2, 30, 30)
    assert (o.max_outer_iterations, o.cg_max_iterations, o.cg_check_interval) == (1000, 100000, 4)
    assert (o.averaging, o.normalizer, o.precision) == (0, 0, 0)
    assert si.RunOptions().to_c().tolerance == o.tolerance


@pytest.mark.parametrize("kw,msg", [
    (dict(tolerance=0.0), "tolerances must be positive"),
    (dict(coarse_tolerance=-1.0), "tolerances must be positive"),
    (dict(levels=0), "levels must be >= 1"),
    (dict(block_size=0), "block_size must be positive"),
    (dict(alpha=float("inf")), "alpha must be finite"),
    (dict(local=si.SolverConfig(0.0, 30, 30)), "tolerance must be positive"),
    (dict(local=si.SolverConfig(1e-2, -1, 30)), "max_iterations must be non-negative"),
    (dict(local=si.SolverConfig(1e-2, 30, 0)), "residual_check_interval must be >= 1"),
])
def test_option_validation_messages(kw, msg):
    lib = L.load()
    o = si.RunOptions(**kw).to_c()
    st = lib.si_validate_options(int(si.Method.MultilevelOras), C.byref(o))
    assert st == L.SI_ERR_INVALID_ARGUMENT
    assert msg in lib.si_last_error().decode()


def test_every_method_validates():
    lib = L.load()
    o = si.RunOptions().to_c()
    for m in si.Method:
        assert lib.si_validate_options(int(m), C.byref(o)) == L.SI_OK
    assert lib.si_validate_options(7, C.byref(o)) == L.SI_ERR_INVALID_ARGUMENT


# ------------------------------------------------------------- partition
def test_partition_uhd_counts():
    """partition_test.cpp:11-16, acceptance_test.cpp:102-108."""
    p = si.partition_domain(3840, 2160, 32, 6)
    assert (p.blocks_x, p.blocks_y, p.size()) == (148, 83, 12284)
    assert p.size() * 3 == 36852


def test_partition_single_block_and_shift():
    """partition_test.cpp:18-38."""
    for ov in (0, 1, 6, 31):
        p = si.partition_domain(32, 32, 32, ov)
        sd = p.subdomains[0]
        assert p.size() == 1 and (sd.x0, sd.y0, sd.own_x1, sd.own_y1) == (0, 0, 32, 32)
    p = si.partition_domain(50, 32, 32, 6)
    assert p.blocks_x == 2 and p.subdomains[0].x0 == 0 and p.subdomains[1].x0 == 18


@pytest.mark.parametrize("args,msg", [((64, 64, 16, 16), "overlap must be smaller"),
                                      ((64, 64, 16, 20), "overlap must be smaller"),
                                      ((64, 64, 16, -1), "overlap must be non-negative"),
                                      ((10, 64, 16, 4), "exceeds image dimensions"),
                                      ((64, 10, 16, 4), "exceeds image dimensions"),
                                      ((64, 64, 0, 0), "block_size must be positive")])
def test_partition_rejects_bad_configurations(args, msg):
    """partition_test.cpp:40-46."""
    with pytest.raises(si.InvalidArgument, match=msg):
        si.partition_domain(*args)


def test_partition_tiles_and_ties(oracle):
    """partition_test.cpp:48-89: owned rectangles tile exactly; ties to the
    lower block; anchors identical to the oracle's partition_axis."""
    rng = np.random.default_rng(7)
    for _ in range(60):
        w, h = (int(v) for v in rng.integers(8, 201, 2))
        block = int(rng.integers(2, min(w, h) + 1))
        ov = int(rng.integers(0, block))
        p = si.partition_domain(w, h, block, ov)
        cover = np.zeros((h, w), np.int32)
        for sd in p.subdomains:
            assert sd.x0 <= sd.own_x0 < sd.own_x1 <= sd.x0 + sd.width
            assert sd.y0 <= sd.own_y0 < sd.own_y1 <= sd.y0 + sd.height
            cover[sd.own_y0:sd.own_y1, sd.own_x0:sd.own_x1] += 1
        assert (cover == 1).all()
        ax, ex = oracle.oracle_partition_axis(w, block, ov)
        assert [p.subdomains[k].x0 for k in range(p.blocks_x)] == ax
        assert [p.subdomains[k].own_x1 for k in range(p.blocks_x)] == ex
    p = si.partition_domain(9, 5, 5, 1)
    assert p.subdomains[0].own_x1 == 5 and p.subdomains[1].own_x0 == 5


def test_clamped_partition():
    p = si.clamped_partition(3, 1, 32, 6)
    assert (p.block_size, p.overlap, p.size()) == (1, 0, 3)


# ------------------------------------------------------------- generators
def test_random_mask_exact_count_and_errors():
    m = si.random_mask(100, 37, 0.05, 3)
    assert m.known_count() == round(0.05 * 3700)
    with pytest.raises(si.InvalidArgument):
        si.random_mask(10, 10, 0.0, 1)
    with pytest.raises(si.InvalidArgument):
        si.random_mask(10, 10, 1.5, 1)
    assert si.random_mask(4, 4, 1.0, 9).known_count() == 16


def test_synthetic_image_range():
    f = si.synthetic_test_image(64, 48, 3, 5)
    for c in range(3):
        assert abs(f.data[c].min() - 0.05) < 1e-12 and abs(f.data[c].max() - 0.95) < 1e-12


def test_psnr_host_helper():
    a = si.ImageBuffer(8, 8, 2, 0.5)
    b = si.ImageBuffer(8, 8, 2, 0.5)
    assert si.psnr(a, b) == float("inf")
    b.data[0, 0, 0] = 0.6
    mse = (255 * 0.1) ** 2 / 64 / 2
    assert si.psnr(a, b) == pytest.approx(10 * np.log10(255 ** 2 / mse), rel=1e-12)


def test_no_device_fails_loudly():
    """Without a GPU the product path raises; it never falls back to the CPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(si.SolverError, match="no CUDA device"):
        si.Solver(0)


def test_cpp_wrapper_header_compiles(tmp_path):
    """include/schwarz_b200.hpp (the C++ drop-in for run_method) compiles and links."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "schwarz_b200.hpp"\n'
                   'int main(){ namespace sb = schwarz_b200;\n'
                   '  auto f = sb::synthetic_test_image(16, 16, 1, 1);\n'
                   '  auto m = sb::random_mask(16, 16, 0.2, 2);\n'
                   '  sb::RunOptions o; (void)o; (void)f; (void)m;\n'
                   '  sb::DensifyOptions d; (void)d;\n'
                   '  auto (*dens)(const sb::ImageBuffer&, double, uint64_t, const sb::DensifyOptions&,\n'
                   '              sb::Context&) = &sb::voronoi_densify; (void)dens;\n'
                   '  auto (*asg)(const sb::InpaintingMask&, sb::Context&) = &sb::assign_nearest_site;\n'
                   '  auto (*bat)(sb::Method, const std::vector<std::pair<const sb::ImageBuffer*,\n'
                   '              const sb::InpaintingMask*>>&, const sb::RunOptions&,\n'
                   '              sb::Context&) = &sb::run_batch; (void)bat;\n'
                   '  (void)asg; return 0; }\n')
    out = subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src),
                          L.lib_path(), "-o", str(tmp_path / "t"),
                          f"-Wl,-rpath,{os.path.dirname(L.lib_path())}"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    run = subprocess.run([str(tmp_path / "t")], capture_output=True, text=True)
    assert run.returncode == 0, run.stderr


def test_batch_outputs_are_validated_before_the_abi():
    """run_batch / run_pnm_batch hand raw pointers to the library: a short
    list, a wrong shape/dtype or a non-contiguous view must raise first."""
    from paper_2110_03946_b200.api import _require_outputs
    good = [np.empty((3, 4, 5)) for _ in range(2)]
    _require_outputs(good, 2, (3, 4, 5), np.float64, "run_batch")
    with pytest.raises(si.InvalidArgument):
        _require_outputs(good[:1], 2, (3, 4, 5), np.float64, "run_batch")
    with pytest.raises(si.InvalidArgument):
        _require_outputs([good[0], np.empty((3, 4, 4))], 2, (3, 4, 5), np.float64, "run_batch")
    with pytest.raises(si.InvalidArgument):
        _require_outputs([good[0], np.empty((3, 4, 5), np.float32)], 2, (3, 4, 5), np.float64,
                         "run_batch")
    with pytest.raises(si.InvalidArgument):
        _require_outputs([good[0], np.empty((3, 4, 10))[:, :, ::2]], 2, (3, 4, 5), np.float64,
                         "run_batch")
    with pytest.raises(si.InvalidArgument):
        _require_outputs([np.empty((4, 5, 3), np.uint8)], 1, (4, 5, 3), np.float64, "run_pnm_batch")


def test_cpp_dropin_types_and_messages(tmp_path):
    """C++20 drop-in (include/schwarz_b200.hpp): the reference's type members
    (ImageBuffer::channel as std::span, InpaintingMask::known_count/density,
    image.hpp:44-93), method names (methods.hpp:15-40) and the exact
    std::invalid_argument messages of random_mask (masks.hpp:26-31),
    require_same_grid (image.hpp:96-99) and channel(); host-only calls."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include <span>
#include "schwarz_b200.hpp"
namespace sb = schwarz_b200;
template <class F> void expect(F&& f) {
  try { f(); std::printf("no-throw\n"); }
  catch (const std::invalid_argument& e) { std::printf("%s\n", e.what()); }
}
int main() {
  sb::ImageBuffer f(5, 4, 2, 0.5);
  std::span<double> c1 = f.channel(1);
  c1[3] = 2.0;
  std::printf("%zu %g %g\n", c1.size(), f.at(3, 0, 1), f.channel(0)[0]);
  auto m = sb::random_mask(5, 4, 0.25, 3);
  std::printf("%zu %.3f\n", m.known_count(), m.density());
  std::printf("%s %d\n", sb::method_name(sb::parse_method("mloras")),
              (int)sb::is_multilevel(sb::Method::MultilevelCg));
  expect([] { sb::random_mask(0, 4, 0.5, 1); });
  expect([] { sb::random_mask(4, 4, 1.5, 1); });
  expect([] { sb::random_mask(4, 4, 0.01, 1); });
  expect([&] { sb::require_same_grid(f, sb::InpaintingMask(4, 4)); });
  expect([&] { (void)f.channel(2); });
  expect([] { sb::parse_method("foo"); });
  return 0;
}
''')
    exe = tmp_path / "t"
    out = subprocess.run(["g++", "-std=c++20", "-Wall", "-I", os.path.join(ROOT, "include"),
                          str(src), L.lib_path(), "-o", str(exe),
                          f"-Wl,-rpath,{os.path.dirname(L.lib_path())}"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True)
    assert run.returncode == 0, run.stderr
    lines = run.stdout.strip().splitlines()
    assert lines[0] == "20 2 0.5"
    assert lines[1] == "5 0.250"
    assert lines[2] == "mloras 1"
    assert lines[3:] == ["random_mask: dimensions must be positive",
                         "random_mask: density must lie in (0, 1]",
                         "random_mask: density rounds to zero known pixels",
                         "image and mask dimensions differ",
                         "ImageBuffer::channel: index out of range",
                         "unknown method 'foo' (expected cg, mlcg, ras, oras or mloras)"]
