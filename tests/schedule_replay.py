"""numpy replay of the GPU schedule (K1 blocks -> K2 levels -> K3 root).

Mirrors paper_2411_07351_b200/csrc/kernels.cu step for step on the host,
including K1's row tiles of S rows with the table-derived halo, so the CPU
tests prove the integer schedule tables (plan.cpp) bit-exact against the
oracle before any CUDA runs.  Test helper only.
"""
import numpy as np


def replay(cols: np.ndarray, sched: dict, S: int) -> np.ndarray:
    """cols[x, y] = working column x, row y (W x H).  Returns OUT_0[t, s]."""
    W, H = cols.shape
    S = min(S, H)
    bufs = [np.zeros((W, H), cols.dtype), np.zeros((W, H), cols.dtype)]
    for x0, shape, depth in sched["blocks"]:
        sh = sched["shapes"][shape]
        wb, steps, halo = sh["width"], sh["steps"], sh["halo"]
        offs, ops = sh["step_offset"], sh["ops"]
        R = S + halo
        for s0 in range(0, H, S):
            rows = (s0 + np.arange(R)) % H
            cur = cols[x0:x0 + wb][:, rows].copy()  # depth `steps` values
            for k in range(steps):
                nxt = np.zeros_like(cur)
                for dst, a, b, r, extra in ops[offs[k]:offs[k + 1]]:
                    n = S + extra
                    assert n <= R and (b < 0 or r + n <= R), "op reads outside the loaded window"
                    nxt[dst, :n] = cur[a, :n] + cur[b, r:r + n] if b >= 0 else cur[a, :n]
                cur = nxt
            m = min(S, H - s0)
            bufs[depth & 1][x0:x0 + wb, s0:s0 + m] = cur[:, :m]
    for lvl in sched["levels"]:
        d = lvl["depth"]
        src, dst = bufs[(d + 1) & 1], bufs[d & 1]
        for t, a, b, r in lvl["ops"]:
            assert 0 <= r < H
            dst[t] = src[a] + np.roll(src[b], -r)
    return bufs[0]


def working_cols(img: np.ndarray, q: int) -> np.ndarray:
    """COLS[x][y] of quadrant q for a row-major (h, w) image."""
    if q == 0:
        return img.T.copy()
    if q == 1:
        return img[:, ::-1].T.copy()
    if q == 2:
        return img.copy()
    return img[::-1, :].copy()
