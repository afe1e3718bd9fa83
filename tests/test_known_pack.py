"""Host-side known-sample packing (si_pack_known_samples, host_copy.h): the
upload format of the host entries.  Host only, no device."""
import numpy as np
import pytest

import paper_2110_03946_b200 as si


def numpy_pack(f, known):
    k = known.reshape(-1) != 0
    counts = np.add.reduceat(k.astype(np.int64), np.arange(0, k.size, si.api.KNOWN_TILE))
    tiles = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint32)
    return tiles, f.reshape(f.shape[0], -1)[:, k]


@pytest.mark.parametrize("w,h,c,density,seed", [
    (333, 211, 3, 0.04, 1),     # tails: w*h not a multiple of 8 or of the tile
    (64, 64, 1, 0.0, 2),        # nothing known
    (97, 13, 2, 1.0, 3),        # everything known
    (4096, 3, 3, 0.02, 4),      # exactly three tiles
    (1, 1, 1, 1.0, 5),
    (517, 389, 5, 0.3, 6),
])
def test_pack_matches_numpy(w, h, c, density, seed):
    rng = np.random.default_rng(seed)
    f = si.ImageBuffer(data=rng.standard_normal((c, h, w)))
    known = (rng.random((h, w)) < density).astype(np.uint8)
    # any nonzero byte marks a known pixel (InpaintingMask::known)
    known *= rng.integers(1, 256, (h, w), dtype=np.uint8)
    m = si.InpaintingMask(known=known)
    tiles, vals = si.pack_known_samples(f, m)
    t_ref, v_ref = numpy_pack(f.data, known)
    assert np.array_equal(tiles, t_ref)
    assert np.array_equal(vals, v_ref)


def test_pack_ignores_unknown_values():
    """NaN / Inf at unknown pixels never reach the upload (build_pyramid
    zeroes them, multilevel.hpp:84-88)."""
    f = si.synthetic_test_image(100, 90, 3, 7)
    m = si.random_mask(100, 90, 0.05, 11)
    f.data[:, m.known == 0] = np.nan
    _, vals = si.pack_known_samples(f, m)
    assert np.isfinite(vals).all()
