"""CPU compute backend for the stripe orchestrator (tests only): numpy + the
C oracle, same interface as stripes.DeviceBackend."""
import numpy as np

from oracle import pyoracle as P
import paper_2110_03946_b200 as si


class OracleBackend:
    def copy(self, a):
        return np.array(a, copy=True)

    def ingest(self, f, mask):
        b = np.where(mask[None] != 0, f, 0.0)
        return b, int(np.count_nonzero(mask))

    def restrict(self, mask, vals, averaging):
        return P.oracle_restrict(mask, vals, averaging)

    def prolong_snap(self, coarse, fmask, fvals):
        c, fh, fw = fvals.shape
        out = np.stack([P.oracle_prolongate(coarse[k], fw, fh) for k in range(c)])
        return np.where(fmask[None] != 0, fvals, out)

    def residual_rows(self, mask, u, b, row0, row1, mode=0):
        if mode == 1:
            return np.array([np.sum(b[k, row0:row1] ** 2) for k in range(b.shape[0])])
        c, h, w = u.shape
        out = []
        for k in range(c):
            uk = u[k]
            s = np.zeros((h, w))
            deg = np.zeros((h, w))
            s[:, 1:] += uk[:, :-1]; deg[:, 1:] += 1
            s[:, :-1] += uk[:, 1:]; deg[:, :-1] += 1
            s[1:, :] += uk[:-1, :]; deg[1:, :] += 1
            s[:-1, :] += uk[1:, :]; deg[:-1, :] += 1
            au = np.where(mask != 0, uk, deg * uk - s)
            r = b[k] - au
            out.append(np.sum(r[row0:row1] ** 2))
        return np.array(out)

    def sweep_rows(self, mask, b, u_old, u_new, block, overlap, by0, by1, flavour, opts):
        full, fails, its = P.oracle_sweep(mask, b, u_old, block, overlap, flavour=flavour,
                                          alpha=opts.alpha)
        part = si.partition_domain(u_old.shape[2], u_old.shape[1], block, overlap)
        lo = part.subdomains[by0 * part.blocks_x].own_y0
        hi = part.subdomains[(by1 - 1) * part.blocks_x].own_y1
        u_new[:, lo:hi, :] = full[:, lo:hi, :]
        return 0, 0
