"""numpy replay of the GPU schedule (K1 blocks -> K2 levels -> K3 root).

Mirrors paper_2411_07351_b200/csrc/kernels.cu step for step on the host,
including K1's row tiles of S rows with the table-derived halo, so the CPU
tests prove the integer schedule tables (plan.cpp) bit-exact against the
oracle before any CUDA runs.  Test helper only.
"""
import numpy as np


def replay(cols: np.ndarray, sched: dict, S: int, pass_S: int | None = None, pairs: bool = False) -> np.ndarray:
    """cols[x, y] = working column x, row y (W x H).  Returns OUT_0[t, s].
    S = K1 row tile; pass_S = K2 row tile (default: H); pairs: run the
    level-pair programs (the 4-byte K2 path) instead of one level per step."""
    W, H = cols.shape
    S = min(S, H)
    PS = min(pass_S or H, H)
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
            bufs[0][x0:x0 + wb, s0:s0 + m] = cur[:, :m]  # K1 = pass 0 -> buffer 0
    if sched["root_is_block"]:
        return bufs[0]
    passes = sched["passes"]
    result = np.zeros((W, H), cols.dtype)
    for p, ps in enumerate(passes):
        ps = _as_unit_program(ps) if pairs else _terms_program(ps)
        src = bufs[p & 1]
        dst = result if p == len(passes) - 1 else bufs[(p + 1) & 1]
        written = np.zeros(W, bool)
        for lb, lc, sb, nsteps, stb, stc, nslots, max_ext in ps["tiles"]:
            for s0 in range(0, H, PS):
                sm = {}
                for gcol, slot, off, ext in ps["loads"][lb:lb + lc]:
                    sm[slot] = src[gcol][(s0 + off + np.arange(PS + ext)) % H]
                for k in range(nsteps):
                    step = ps["ops"][ps["step_offs"][sb + k]:ps["step_offs"][sb + k + 1]]
                    reads = {slot for o in step for slot, _ in o[2]}
                    writes = [o[0] for o in step]
                    assert len(set(writes)) == len(writes) and not (set(writes) & reads), "slot reuse within a step"
                    new = {}
                    for d, ext, terms, *_ in step:
                        n = PS + ext
                        assert all(off >= 0 and off + n <= len(sm[slot]) for slot, off in terms), "window overrun"
                        acc = sm[terms[0][0]][terms[0][1]:terms[0][1] + n].copy()
                        for slot, off in terms[1:]:
                            acc = acc + sm[slot][off:off + n]
                        new[d] = acc
                    assert max(writes, default=-1) < nslots
                    sm.update(new)
                m = min(PS, H - s0)
                for slot, gcol in ps["stores"][stb:stb + stc]:
                    dst[gcol, s0:s0 + m] = sm[slot][:m]
                    written[gcol] = True
        assert written.all(), "a pass did not write every column"
    return result


def _as_unit_program(ps: dict) -> dict:
    return dict(ps["pairs"], loads=ps["loads"])


def _terms_program(ps: dict) -> dict:
    """One-level ops [dst, a, b, ad, bd, ext] as [dst, ext, terms]."""
    ops = [[d, ext, [[a, ad]] + ([[b, bd]] if b >= 0 else [])] for d, a, b, ad, bd, ext in ps["ops"]]
    return dict(ps, ops=ops)


def working_cols(img: np.ndarray, q: int) -> np.ndarray:
    """COLS[x][y] of quadrant q for a row-major (h, w) image."""
    if q == 0:
        return img.T.copy()
    if q == 1:
        return img[:, ::-1].T.copy()
    if q == 2:
        return img.copy()
    return img[::-1, :].copy()
