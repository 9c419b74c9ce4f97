"""GPU parity at BASELINE.json's full chunk sizes through size-independent
properties:

* C3 — one GPT-3-65B block (12*8192^2 = 805,306,368 params): the streamed
  step (fy_pipeline_*, master/m/v in pinned host memory, 12 B/param H2D and
  14 B/param D2H) equals the device-resident step on the same inputs, bit for
  bit, over two consecutive steps; three windows are also checked against the
  CPU oracle (Adam is elementwise, so a window of the input maps to the same
  window of the output).
* C4 — one GPT-3-175B block (12*12288^2 = 1,811,939,328 params) sharded
  across 8 simulated ranks (fy_shard_range slices, fused all-gather epilogue
  into 8 full-param buffers) equals the single-launch step on the whole
  chunk, bit for bit, in every rank's buffer, and the CPU oracle in windows
  at the chunk's ends and straddling every rank boundary.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_65B = 12 * 8192 * 8192
N_175B = 12 * 12288 * 12288
WINDOW = 1 << 20


def _states(n, dev, seed):
    g = torch.Generator(device=dev)
    g.manual_seed(20240817 + seed)
    st = torch.empty(3 * n, device=dev)
    st[:n].normal_(0, 0.02, generator=g)
    st[n:2 * n].normal_(0, 1e-3, generator=g)
    st[2 * n:].normal_(0, 1e-3, generator=g).square_()
    grad = (torch.randn(n, device=dev, generator=g) * 1e-3).to(torch.bfloat16)
    return st, grad


def _same_bits(a: torch.Tensor, b: torch.Tensor) -> bool:
    view = torch.int32 if a.element_size() == 4 else torch.int16
    return bool(torch.equal(a.view(view), b.view(view)))


def _oracle_windows(n, st0, grad, st1, param, hp_step, los=None):
    """Windows [0, W), the middle and the last W elements (or `los`) vs the
    oracle."""
    sc = O.scalars(step=hp_step)
    for lo in (los or (0, n // 2 - WINDOW // 2, n - WINDOW)):
        sl = slice(lo, lo + WINDOW)
        mst = st0[:n][sl].cpu().numpy().copy()
        mm = st0[n:2 * n][sl].cpu().numpy().copy()
        vv = st0[2 * n:][sl].cpu().numpy().copy()
        g = grad[sl].cpu().view(torch.int16).numpy().view(np.uint16).copy()
        p = np.zeros(WINDOW, np.uint16)
        O.adamw_step(mst, mm, vv, g, O.BF16, sc, param_out=p)
        for got, ref in ((st1[:n][sl], mst), (st1[n:2 * n][sl], mm), (st1[2 * n:][sl], vv)):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        assert np.array_equal(param[sl].cpu().view(torch.int16).numpy().view(np.uint16), p)


def test_c3_65b_block_streamed_equals_resident(cuda_dev):
    from paper_2403_06504_b200 import optim as F
    n = N_65B
    st, grad = _states(n, cuda_dev, 65)
    st0 = st.clone()                       # initial states (oracle windows)
    h_states = st.cpu().pin_memory()       # streamed copy (pinned host)
    h_param = torch.zeros(n, dtype=torch.bfloat16).pin_memory()
    d_param = torch.empty(n, dtype=torch.bfloat16, device=cuda_dev)
    pipe = F.ChunkPipeline(n, slots=2)
    try:
        for step in (10, 11):
            hp = F.Hparams(step=step)
            # resident: the kernel on HBM states
            F.adamw_chunk(st[:n], st[n:2 * n], st[2 * n:], grad, hp, param_out=d_param)
            # streamed: the pipeline on host states
            pipe.step([dict(n=n, h_states=h_states.data_ptr(), grad=grad.data_ptr(),
                            h_param=h_param.data_ptr())], hp)
            pipe.wait()
            torch.cuda.synchronize()
            assert _same_bits(h_states.to(cuda_dev), st), f"step {step}: states differ"
            assert _same_bits(h_param.to(cuda_dev), d_param), f"step {step}: params differ"
            if step == 10:
                _oracle_windows(n, st0, grad, st, d_param, step)
                del st0
    finally:
        pipe.close()


def test_c4_175b_block_sharded_8_equals_single(cuda_dev):
    from paper_2403_06504_b200 import optim as F
    n, world = N_175B, 8
    st, grad = _states(n, cuda_dev, 175)
    # oracle windows: the chunk's first and last W elements and one window
    # straddling every rank boundary of the 8-way slicing
    bounds = [F.shard_range(n, world, r, 8)[0] for r in range(1, world)]
    los = [0, n - WINDOW] + [b - WINDOW // 2 for b in bounds]
    win0 = {lo: (st[lo:lo + WINDOW].clone(), st[n + lo:n + lo + WINDOW].clone(),
                 st[2 * n + lo:2 * n + lo + WINDOW].clone(), grad[lo:lo + WINDOW].clone()) for lo in los}
    single = st.clone()
    p_single = torch.empty(n, dtype=torch.bfloat16, device=cuda_dev)
    hp = F.Hparams()
    F.adamw_chunk(single[:n], single[n:2 * n], single[2 * n:], grad, hp, param_out=p_single)
    full = [torch.zeros(n, dtype=torch.bfloat16, device=cuda_dev) for _ in range(world)]
    local = torch.empty(n, dtype=torch.bfloat16, device=cuda_dev)
    covered = 0
    for r in range(world):
        off, cnt = F.shard_range(n, world, r, 8)
        assert off == covered
        covered += cnt
        sl = slice(off, off + cnt)
        F.adamw_chunk_gather(st[:n][sl], st[n:2 * n][sl], st[2 * n:][sl], grad[sl], hp,
                             local[sl], [b.data_ptr() + 2 * off for b in full])
    assert covered == n
    torch.cuda.synchronize()
    assert _same_bits(st, single), "sharded states differ from the single launch"
    for r, b in enumerate(full + [local]):
        assert _same_bits(b, p_single), f"rank buffer {r} differs"
    # the sharded result against the CPU oracle in the windows
    sc = O.scalars(step=hp.step)
    for lo, (m0, mm0, vv0, g0) in win0.items():
        mst, mm, vv = (x.cpu().numpy().copy() for x in (m0, mm0, vv0))
        g = g0.cpu().view(torch.int16).numpy().view(np.uint16).copy()
        p = np.zeros(WINDOW, np.uint16)
        O.adamw_step(mst, mm, vv, g, O.BF16, sc, param_out=p)
        sl = slice(lo, lo + WINDOW)
        for got, ref in ((st[:n][sl], mst), (st[n:2 * n][sl], mm), (st[2 * n:][sl], vv)):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), ref.view(np.uint32)), lo
        for b in full:
            assert np.array_equal(b[sl].cpu().view(torch.int16).numpy().view(np.uint16), p), lo


N_HUGE = (1 << 32) + 3 * 2048 + 5  # one chunk past 2^32 elements (60 GB of states + grads)


@pytest.mark.parametrize("path", ["tma", "lsu"])
def test_chunk_past_2pow32_elements(cuda_dev, path):
    """Maximum sizes: one launch over a chunk of 2^32 + 6149 elements (no
    32-bit index may wrap) equals launches over 2^30-element slices of the
    same inputs bit for bit (Adam is elementwise), and windows straddling
    2^31 and 2^32 plus the ragged tail equal the CPU oracle."""
    from paper_2403_06504_b200 import optim as F
    from paper_2403_06504_b200._lib import LIB, check
    torch.cuda.empty_cache()  # the other path's 120 GB, still cached by torch
    free, _ = torch.cuda.mem_get_info(cuda_dev)
    if free < 135e9:
        pytest.skip(f"needs ~125 GB of free HBM, {free / 1e9:.0f} GB free")
    n = N_HUGE
    check(LIB.fy_adamw_tune(1, 3, 0) if path == "tma" else LIB.fy_adamw_tune(0, 2, 2))
    try:
        st, grad = _states(n, cuda_dev, 32)
        los = (0, (1 << 31) - WINDOW // 2, n - WINDOW)  # the last window straddles 2^32
        init = {lo: ([st[k * n + lo:k * n + lo + WINDOW].cpu().numpy().copy() for k in range(3)],
                     grad[lo:lo + WINDOW].cpu().view(torch.int16).numpy().view(np.uint16).copy()) for lo in los}
        # float64 reference of the grad sum of squares (before the in-place
        # update overwrites the grads with params), in 2^28-element pieces
        exp_sq = sum(float(grad[lo:lo + (1 << 28)].double().square().sum()) for lo in range(0, n, 1 << 28))
        st2, grad2 = st.clone(), grad.clone()
        hp = F.Hparams(step=7)
        ws = torch.zeros(F.workspace_floats(), device=cuda_dev)
        sq1, sq2 = (torch.zeros(1, dtype=torch.float64, device=cuda_dev) for _ in range(2))
        F.adamw_chunk(st[:n], st[n:2 * n], st[2 * n:], grad, hp, param_out=grad,  # in place
                      grad_sq_sum=sq1, workspace=ws)
        piece = 1 << 30
        for lo in range(0, n, piece):
            hi = min(n, lo + piece)
            F.adamw_chunk(st2[lo:hi], st2[n + lo:n + hi], st2[2 * n + lo:2 * n + hi], grad2[lo:hi], hp,
                          param_out=grad2[lo:hi], grad_sq_sum=sq2, accumulate_sq=lo > 0, workspace=ws)
        torch.cuda.synchronize()
        assert _same_bits(st, st2) and _same_bits(grad, grad2)
        # per-CTA partials are rounded to float once (~6e-8); the per-thread
        # sums must not drift over 2^32 elements (fp32 running sums: 1.5e-5)
        for got in (sq1.item(), sq2.item()):
            assert abs(got - exp_sq) <= 1e-6 * exp_sq, (got, exp_sq)
        del st2, grad2
        sc = O.scalars(step=7)
        for lo, ((mst, mm, vv), g) in init.items():
            p = np.zeros(WINDOW, np.uint16)
            O.adamw_step(mst, mm, vv, g, O.BF16, sc, param_out=p)
            for k, ref in enumerate((mst, mm, vv)):
                got = st[k * n + lo:k * n + lo + WINDOW].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (lo, k)
            assert np.array_equal(grad[lo:lo + WINDOW].cpu().view(torch.int16).numpy().view(np.uint16), p), lo
    finally:
        check(LIB.fy_adamw_tune(1, 0, 0))
