"""CPU: pin the AdamW oracle against torch.optim golden vectors, and the
16-bit codecs against torch's conversions (no GPU needed)."""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden" / "adamw_torch_golden.npz"

# Tolerance: the oracle follows DeepSpeed's op order (explicit
# FMAs, 1/sqrt(1-b2^t) in float, -lr/bc1 in float); torch.optim rounds
# differently (lerp, division by sqrt(bc2), double step size). Each result may
# differ by a few float32 ulps of the *summands*, so the bound is relative to
# the magnitude of the terms that produce it:
RTOL = 1e-6


def _bound(*terms):
    return RTOL * sum(np.abs(t) for t in terms) + 1e-30


def _close(x, ref, bound):
    """Finite entries within `bound`; non-finite entries (fp16 overflow ->
    inf grad -> inf/nan state) must be non-finite in both. (inf vs nan may
    differ: torch's lerp turns an inf moment into nan, DeepSpeed's mul+fma
    keeps it inf — neither is meaningful after an overflow.)"""
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(x), fin)
    with np.errstate(invalid="ignore"):
        return bool(np.all(np.abs(x[fin] - ref[fin]) <= np.broadcast_to(bound, ref.shape)[fin]))


@pytest.mark.parametrize("case", range(4))
def test_oracle_matches_torch_adamw(case):
    g = np.load(GOLD)
    t = f"case{case}"
    kind, adamw, wd, grad_scale, first = g[f"{t}_meta"]
    master, m, v = (g[f"{t}_master0"].copy(), g[f"{t}_m0"].copy(), g[f"{t}_v0"].copy())
    grads = g[f"{t}_grads"]
    for s in range(int(g["steps"])):
        sc = O.scalars(lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=float(wd),
                       step=int(first) + s, adamw_mode=bool(adamw))
        m_old, v_old, p_old = m.copy(), v.copy(), master.copy()
        gbits = np.ascontiguousarray(grads[s])
        O.adamw_step(master, m, v, gbits, O.BF16 if kind == 0 else O.FP16, sc,
                     grad_scale=float(grad_scale))
        tm, tv, tp = g[f"{t}_m{s + 1}"], g[f"{t}_v{s + 1}"], g[f"{t}_master{s + 1}"]
        gf = (torch.from_numpy(gbits.view(np.int16)).view(
            torch.bfloat16 if kind == 0 else torch.float16).float().numpy() * grad_scale)
        geff = gf if adamw else gf + float(wd) * p_old
        with np.errstate(invalid="ignore", over="ignore"):
            bm = _bound(0.9 * m_old, 0.1 * geff)
            bv = _bound(0.95 * v_old, 0.05 * geff * geff)
            upd = np.abs(tp - p_old)
            bp = _bound(p_old, upd) + 4 * RTOL * upd
        assert _close(m, tm, bm), f"m step {s}"
        assert _close(v, tv, bv), f"v step {s}"
        assert _close(master, tp, bp), f"p step {s}"
        # the golden torch trajectory is fed forward (pins drift, not just one step)
        master, m, v = tp.copy(), tm.copy(), tv.copy()


def test_codecs_match_torch():
    rng = np.random.default_rng(7)
    x = np.concatenate([
        rng.normal(0, 1, 20000).astype(np.float32),
        rng.normal(0, 1e-5, 5000).astype(np.float32),
        np.array([0.0, -0.0, np.inf, -np.inf, 65504.0, 65519.9, 65520.0, 1e-8, 6e-8, 3e-8,
                  5.96e-8, 2.98e-8, 1e38, -1e-40, 3.4e38], dtype=np.float32)])
    tb = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    th = torch.from_numpy(x).to(torch.float16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.f32_to_bf16_bits(x), tb)
    assert np.array_equal(O.f32_to_fp16_bits(x), th)
    # decode round trip for every 16-bit pattern (non-NaN)
    allbits = np.arange(65536, dtype=np.uint16)
    dec_b = np.array([O.LIB.oracle_bf16_to_float(int(b)) for b in allbits[::7]], dtype=np.float32)
    ref_b = torch.from_numpy(allbits[::7].view(np.int16)).view(torch.bfloat16).float().numpy()
    ok = ~np.isnan(ref_b)
    assert np.array_equal(dec_b[ok], ref_b[ok])
    dec_h = np.array([O.LIB.oracle_fp16_to_float(int(b)) for b in allbits[::7]], dtype=np.float32)
    ref_h = torch.from_numpy(allbits[::7].view(np.int16)).view(torch.float16).float().numpy()
    ok = ~np.isnan(ref_h)
    assert np.array_equal(dec_h[ok], ref_h[ok])


def test_nan_maps_to_canonical():
    assert O.LIB.oracle_float_to_bf16(float("nan")) == 0x7FFF
    assert O.LIB.oracle_float_to_fp16(float("nan")) == 0x7FFF


def test_omp_equals_scalar():
    rng = np.random.default_rng(3)
    n = 100003
    master = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = (rng.normal(0, 1e-3, n) ** 2).astype(np.float32)
    g = O.f32_to_bf16_bits(rng.normal(0, 1e-3, n).astype(np.float32)) if n < 0 else \
        torch.from_numpy(rng.normal(0, 1e-3, n).astype(np.float32)).to(torch.bfloat16).view(
            torch.int16).numpy().view(np.uint16)
    s = O.scalars()
    a = [x.copy() for x in (master, m, v)]
    b = [x.copy() for x in (master, m, v)]
    pa = np.zeros(n, np.uint16)
    pb = np.zeros(n, np.uint16)
    O.adamw_step(*a, g, O.BF16, s, param_out=pa)
    O.adamw_step_omp(*b, g, O.BF16, s, param_out=pb, threads=4)
    for x, y in zip(a + [pa], b + [pb]):
        assert np.array_equal(x.view(np.uint32) if x.dtype == np.float32 else x,
                              y.view(np.uint32) if y.dtype == np.float32 else y)


TRAJ = Path(__file__).resolve().parent / "golden" / "adamw_trajectory_golden.npz"


def trajectory_check(s, c, old, got, gold, grad_bits):
    """One step of chunk c against torch (fed forward from torch's previous
    state). Two bars (north star: "rel 1e-6 on params and m/v"):
      * every element: within 1e-6 of the magnitude of its summands (_bound);
      * per-element RELATIVE 1e-6 wherever the result is well conditioned
        (condition number <= 4: the summands do not cancel — for m,
        (b1|m_old| + (1-b1)|g|) / |m|; for params, (|p_old| + |upd| cond_m)
        / |p|, since the update inherits m's cancellation); v never cancels,
        so all of v. The well-conditioned share is asserted too.
    Returns the covered fractions."""
    p0, m0, v0 = old
    p, m, v = got
    tp, tm, tv = gold
    gf = (grad_bits.astype(np.uint32) << 16).view(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        cond_m = (0.9 * np.abs(m0) + 0.1 * np.abs(gf)) / np.abs(tm)
        upd = np.abs(tp - p0)
        cond_p = (np.abs(p0) + upd * np.where(np.isfinite(cond_m), cond_m, 1e30)) / np.abs(tp)
        rel = lambda x, r: np.abs(x - r) / np.abs(r)
        assert _close(m, tm, _bound(0.9 * m0, 0.1 * gf)), f"m step {s} chunk {c}"
        assert _close(v, tv, _bound(0.95 * v0, 0.05 * gf * gf)), f"v step {s} chunk {c}"
        assert _close(p, tp, _bound(p0, upd) + 4 * RTOL * upd), f"p step {s} chunk {c}"
        okm, okp = cond_m <= 4, cond_p <= 4
        assert np.all(rel(m, tm)[okm] <= RTOL), f"m rel step {s} chunk {c}"
        assert np.all(rel(p, tp)[okp] <= RTOL), f"p rel step {s} chunk {c}"
        assert np.all(rel(v, tv)[tv != 0] <= RTOL), f"v rel step {s} chunk {c}"
    return okm.mean(), okp.mean()


def oracle_trajectory(counter=True):
    """The oracle over the fixture: per step, every chunk from torch's
    previous state, beta^t from DeepSpeed's step counter (one increment per
    chunk, as DeepSpeedCPUAdam calls adam_update per sub-group)."""
    g = np.load(TRAJ)
    sizes, steps = [int(x) for x in g["sizes"]], int(g["steps"])
    k = O.StepCounter()
    for s in range(steps):
        for c, n in enumerate(sizes):
            if s == 0:
                old = (g[f"c{c}_master0"], np.zeros(n, np.float32), np.zeros(n, np.float32))
            else:
                old = (g[f"c{c}_master{s}"], g[f"c{c}_m{s}"], g[f"c{c}_v{s}"])
            st = [x.copy() for x in old]
            sc = O.scalars_bt(*k.next(s + 1)) if counter else O.scalars(step=s + 1)
            gb = np.ascontiguousarray(g[f"c{c}_grads"][s])
            O.adamw_step(*st, gb, O.BF16, sc)
            yield s, c, old, st, (g[f"c{c}_master{s + 1}"], g[f"c{c}_m{s + 1}"], g[f"c{c}_v{s + 1}"]), gb


def test_oracle_trajectory_with_step_counter_matches_torch():
    cov = [trajectory_check(s, c, old, st, gold, gb) for s, c, old, st, gold, gb in oracle_trajectory()]
    assert np.mean([a for a, _ in cov]) > 0.8 and np.mean([b for _, b in cov]) > 0.99
