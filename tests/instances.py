"""Seeded instances shared by the test modules (tests/support/instances.hpp:20-37)."""
import numpy as np

import paper_2110_03946_b200 as si


def random_instance(width, height, density, channels, seed):
    """synthetic image + uniform random mask, seeds as the reference's tests use them."""
    img = si.synthetic_test_image(width, height, channels, seed)
    min_density = 1.0 / (width * height)
    mask = si.random_mask(width, height, max(density, 1.5 * min_density),
                          (seed ^ 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
    return img, mask


def random_vector(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# BASELINE.json configs: (w, h, channels, density, levels)
C1 = (256, 256, 1, 0.05, 2)
C2 = (1920, 1080, 3, 0.04, 2)
C3 = (3840, 2160, 3, 0.04, 3)


def config_instance(cfg, k=0):
    w, h, c, d, _ = cfg
    return si.synthetic_test_image(w, h, c, 7 + k), si.random_mask(w, h, d, 11 + k)
