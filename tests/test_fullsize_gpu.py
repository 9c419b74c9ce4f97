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
  chunk, bit for bit, in every rank's buffer.
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


def _oracle_windows(n, st0, grad, st1, param, hp_step):
    """Windows [0, W), the middle and the last W elements vs the oracle."""
    sc = O.scalars(step=hp_step)
    for lo in (0, n // 2 - WINDOW // 2, n - WINDOW):
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
