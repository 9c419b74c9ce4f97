"""GPU: the whole-iteration executor (fy_graph_execute / offsim_execute) on
the GPT-2-small-shaped config C1 (12 blocks x 12*768^2 params): every task
of the planner's graph runs on real engines; the executed trace must pass the
UNCHANGED check_trace_invariants, every swapped activation / checkpoint must
round-trip bit-exactly, the per-chunk Adam results must equal the CPU oracle
bit-for-bit, and the physically moved bytes must equal the mapped graph's."""
import numpy as np
import pytest
import torch

from exec_api import execute, graph_execute, scenario
from oracle import oracle as O

pytestmark = pytest.mark.gpu

L, H = 12, 768
N = 12 * H * H
RATE = 1.4e15  # synthetic compute at the measured sustained bf16 rate


def _chunks(dev, seed=0):
    chunks, ref = [], []
    for k in range(L):
        rng = np.random.default_rng(20240817 + seed + k)
        st = np.empty(3 * N, np.float32)
        st[:N] = rng.normal(0, 0.02, N)
        st[N:2 * N] = rng.normal(0, 1e-3, N)
        st[2 * N:] = rng.normal(0, 1e-3, N) ** 2
        g = torch.from_numpy(rng.normal(0, 1e-3, N).astype(np.float32)).to(torch.bfloat16)
        hs = torch.from_numpy(st.copy()).pin_memory()
        hp = torch.zeros(N, dtype=torch.bfloat16).pin_memory()
        dg = g.to(dev)
        chunks.append(dict(n=N, h_states=hs.data_ptr(), grad=dg.data_ptr(), h_param=hp.data_ptr(),
                           _keep=(hs, hp, dg)))
        ref.append((st, g.view(torch.int16).numpy().view(np.uint16).copy()))
    return chunks, ref


def _oracle_check(chunks, ref, s, step=10):
    sc = O.scalars(step=step)
    sq = 0.0
    for c, (st, g) in zip(chunks, ref):
        m, mo, v = st[:N].copy(), st[N:2 * N].copy(), st[2 * N:].copy()
        p = np.zeros(N, np.uint16)
        s_, _ = O.adamw_step(m, mo, v, g, O.BF16, sc, param_out=p)
        sq += s_
        hs, hp, _ = c["_keep"]
        got = hs.numpy()
        assert np.array_equal(got[:N].view(np.uint32), m.view(np.uint32)), "master"
        assert np.array_equal(got[N:2 * N].view(np.uint32), mo.view(np.uint32)), "m"
        assert np.array_equal(got[2 * N:].view(np.uint32), v.view(np.uint32)), "v"
        assert np.array_equal(hp.view(torch.int16).numpy().view(np.uint16), p), "params"
    assert abs(s["optimizer"]["grad_sq_sum"] - sq) <= 2e-7 * sq


def _failing(s):
    return None if s is None else [e for e in s["invariants"] if not e["pass"]]


def _inv(s):
    return {e["name"]: (e["pass"], e["detail"]) for e in s["invariants"]}


@pytest.mark.parametrize("launch", ["graph", "stream"])
def test_c1_overlapped_host_tier_matches_oracle(cuda_dev, launch):
    """Both launch modes: the iteration captured once into a CUDA graph (the
    default) and issued task by task on the lane streams."""
    chunks, ref = _chunks(cuda_dev)
    st, s, err = graph_execute(scenario(), {"tier": "host", "compute_rate": RATE, "launch": launch}, chunks)
    assert st == 0, (err, _failing(s))
    assert s["launch"] == launch
    assert s["all_invariants_pass"], s["invariants"]
    assert s["swap_mismatches"] == 0 and s["swap_checks"] == L  # one checkpoint per block
    pb = s["physical_bytes"]
    assert pb["h2d/opt_states"] == 12 * N * L and pb["d2h/opt_states"] == 12 * N * L
    assert pb["d2h/params"] == 2 * N * L
    assert "file_read/opt_states" not in pb
    _oracle_check(chunks, ref, s)


def test_c1_b128_swapped_layers_round_trip(cuda_dev):
    # b=128: the planner swaps 13 linear_4htoh activations (coefficient 0.139)
    st, s, _, err = execute(scenario(batch=128), {"tier": "host", "compute_rate": RATE})
    assert st == 0, (err, _failing(s))
    assert s["all_invariants_pass"], s["invariants"]
    assert s["swap_checks"] == L + 13 and s["swap_mismatches"] == 0
    assert s["physical_bytes"]["d2h/activations"] == s["reference_bytes"]["link_g2c/activations"]
    assert s["physical_bytes"]["h2d/activations"] == s["reference_bytes"]["link_c2g/activations"]


@pytest.mark.parametrize("launch", ["graph", "stream"])
def test_c1_file_tier_checkpoints_on_ssd(cuda_dev, tmp_path, launch):
    # cpu_mem 1 GB forces the planner's checkpoint placement to SSD; the file
    # IO runs as host nodes of the captured graph / host functions on the lane
    sc = scenario(hardware='{"preset": "a100-12ssd", "cpu_mem": 1000000000}')
    chunks, ref = _chunks(cuda_dev, seed=100)
    st, s, err = graph_execute(sc, {"tier": "file", "file_dir": str(tmp_path),
                                    "compute_rate": RATE, "launch": launch}, chunks)
    assert st == 0, (err, _failing(s))
    assert s["launch"] == launch
    assert s["checkpoint_location"] == "ssd"
    assert s["all_invariants_pass"], s["invariants"]
    assert s["swap_mismatches"] == 0 and s["swap_checks"] == L
    pb, rb = s["physical_bytes"], s["reference_bytes"]
    assert pb["file_read/opt_states"] == rb["link_ssd/opt_states"] / 2
    assert pb["file_write/opt_states"] == rb["link_ssd/opt_states"] / 2
    assert pb["file_write/activations"] + pb["file_read/activations"] == rb["link_ssd/activations"]
    _oracle_check(chunks, ref, s)


def test_pipelined_file_tier_grads_round_trip(cuda_dev, tmp_path):
    chunks, ref = _chunks(cuda_dev, seed=200)
    st, s, err = graph_execute(scenario(variant="pipelined"),
                               {"tier": "file", "file_dir": str(tmp_path), "compute_rate": RATE},
                               chunks)
    assert st == 0, (err, _failing(s))
    inv = _inv(s)
    assert inv["gradient-ssd-roundtrip"][0], inv["gradient-ssd-roundtrip"]
    assert s["all_invariants_pass"], s["invariants"]
    _oracle_check(chunks, ref, s)


def test_serial_file_tier(cuda_dev, tmp_path):
    st, s, _, err = execute(scenario(variant="serial"),
                            {"tier": "file", "file_dir": str(tmp_path), "compute_rate": RATE})
    inv = _inv(s)
    # a real trace has launch gaps, so only the DES can make makespan equal
    # the duration sum; everything else must hold
    for name, (ok, detail) in inv.items():
        if name != "makespan-equals-duration-sum":
            assert ok, (name, detail)
    assert inv["strictly-serial"][0]


def test_c1_gemm_compute_mode_matches_oracle(cuda_dev):
    # fwd/bwd compute as real cuBLAS bf16 GEMMs: the optimizer overlaps
    # tensor-core work; the Adam results must not change by a bit
    chunks, ref = _chunks(cuda_dev, seed=300)
    st, s, err = graph_execute(scenario(), {"tier": "host", "compute_mode": "gemm"}, chunks)
    assert st == 0, (err, _failing(s))
    assert s["all_invariants_pass"], s["invariants"]
    assert s["hw_exec"]["gpu_tput"] > 1e14  # measured GEMM rate, not the preset's
    _oracle_check(chunks, ref, s)


@pytest.mark.parametrize("placement,tier", [("auto", "host"), ("ssd", "file")])
def test_swap_only_subgraph(cuda_dev, tmp_path, placement, tier):
    # BASELINE config 5 path: only the activation-swap tasks, first 3 blocks
    # of C1 at b=128. The planner swaps 13 layers: the 12 linear_4htoh
    # (priority queue) + block 0's linear_qkv -> 4 activations + 3
    # checkpoints in blocks 0-2
    opts = {"tier": tier, "swap_only": True, "max_blocks": 3, "placement": placement,
            "file_dir": str(tmp_path)}
    st, s, _, err = execute(scenario(batch=128), opts)
    assert st == 0, (err, _failing(s))
    assert s["all_invariants_pass"], s["invariants"]
    assert s["swap_checks"] == 4 + 3 and s["swap_mismatches"] == 0
    rb, pb = s["reference_bytes"], s["physical_bytes"]
    assert pb["d2h/activations"] == rb["link_g2c/activations"]
    assert pb["h2d/activations"] == rb["link_c2g/activations"]
    if placement == "ssd":
        assert s["io_engine"] in ("io_uring", "pread/pwrite")
        assert pb["file_write/activations"] + pb["file_read/activations"] == rb["link_ssd/activations"]
    assert "h2d/opt_states" not in pb  # no optimizer state touched


def test_file_tier_bounded_ring_matches_host_tier(cuda_dev, tmp_path):
    # The SSD tier proper: states/params/weights/activations staged through
    # 2-slot pinned rings; the final states (read back from the files) must
    # equal the host-tier run's bit for bit, with far less pinned memory.
    sc = scenario(hardware='{"preset": "a100-12ssd", "cpu_mem": 1000000000}')
    st, host, _, err = execute(sc, {"tier": "host", "compute_rate": RATE, "checksum_states": True,
                                    "seed": 5})
    assert st == 0, (err, _failing(host))
    for depth in (2, "auto"):
        st, ring, _, err = execute(sc, {"tier": "file", "file_dir": str(tmp_path), "host_ring": depth,
                                        "compute_rate": RATE, "checksum_states": True, "seed": 5})
        assert st == 0, (err, _failing(ring))
        assert ring["all_invariants_pass"], ring["invariants"]
        assert ring["swap_mismatches"] == 0 and ring["swap_checks"] == L
        assert ring["state_checksum"] == host["state_checksum"] != 0
        if depth == 2:
            assert ring["host_ring"] == {"states": 2, "params": 2, "weights": 2, "acts": 2}
            assert ring["pinned_host_bytes"] < host["pinned_host_bytes"] / 2
        else:  # depths from the reference schedule's windows
            assert ring["host_ring"]["states"] == 3 and ring["host_ring"]["weights"] >= 2
        io = ring["io_requests"]
        if ring["io_engine"] == "io_uring" and io["registered_bytes"] > 0:
            # every file request's host side is a registered ring slot
            assert io["fixed"] > 0 and io["plain"] == 0, io
    # striped over three directories (one per SSD): the same states
    dirs = [str(tmp_path / f"ssd{i}") for i in range(3)]
    st, striped, _, err = execute(sc, {"tier": "file", "file_dir": dirs, "host_ring": 2,
                                       "compute_rate": RATE, "checksum_states": True, "seed": 5})
    assert st == 0, (err, _failing(striped))
    assert striped["all_invariants_pass"] and striped["swap_mismatches"] == 0
    assert striped["file_devices"] == 3 and striped["state_checksum"] == host["state_checksum"]
    # registration off: the same result through plain requests
    st, plain, _, err = execute(sc, {"tier": "file", "file_dir": str(tmp_path), "host_ring": 2,
                                     "compute_rate": RATE, "checksum_states": True, "seed": 5,
                                     "fixed_buffers": False})
    assert st == 0, (err, _failing(plain))
    assert plain["state_checksum"] == host["state_checksum"]
    assert plain["io_requests"]["fixed"] == 0 and plain["io_requests"]["registered_bytes"] == 0


def test_gemm_dataflow_grads_feed_the_optimizer(cuda_dev):
    """compute_mode "gemm_dataflow": every layer's backward wgrad GEMM
    (X^T dY, cuBLAS bf16) writes its block's gradient buffer, and the fused
    optimizer consumes exactly those gradients: its accumulated grad sum of
    squares equals the independently computed blocks x sum_j |dW_j|^2; all
    reference invariants hold on the real trace."""
    sc = scenario(layers=6, batch=2, seq=512)
    st, summ, _, err = execute(sc, {"tier": "host", "compute_mode": "gemm_dataflow"})
    assert st == 0, err
    assert summ["all_invariants_pass"], summ["invariants"]
    opt = summ["optimizer"]
    exp = opt["expected_grad_sq_sum"]
    assert exp > 0 and opt["nonfinite"] == 0
    assert abs(opt["grad_sq_sum"] - exp) <= 1e-5 * exp
    # and the synthetic-grad mode does not match it (the grads really changed)
    st2, summ2, _, err2 = execute(sc, {"tier": "host", "compute_mode": "gemm"})
    assert st2 == 0, err2
    assert abs(summ2["optimizer"]["grad_sq_sum"] - exp) > 1e-3 * exp


@pytest.mark.parametrize("tier,R", [("host", 3), ("file", 3), ("host", "auto")])
def test_resident_groups_same_states_fewer_bytes(cuda_dev, tmp_path, tier, R):
    """resident_groups keeps g0..g2's optimizer states in HBM for the run:
    the final states (checksum over every chunk, written back to the tier)
    equal those of the all-streamed run bit for bit, the state bytes moved
    drop by 2 x 12N per resident group, and the invariants hold."""
    sc = scenario(layers=6, batch=2, seq=512)
    base = {"tier": tier, "checksum_states": True, "seed": 7}
    if tier == "file":
        base.update(file_dir=str(tmp_path))
    st0, s0, _, e0 = execute(sc, base)
    st1, s1, _, e1 = execute(sc, {**base, "resident_groups": R})
    assert st0 == 0 and st1 == 0, (e0, e1)
    assert s1["all_invariants_pass"], s1["invariants"]
    assert s1["state_checksum"] == s0["state_checksum"] != 0
    r = 6 if R == "auto" else R  # auto: the C1-sized slice's 6 groups all fit in HBM
    assert s1["resident_groups"] == r
    n = 12 * 768 * 768
    pb0, pb1 = s0["physical_bytes"], s1["physical_bytes"]
    assert pb1.get("h2d/opt_states", 0) == pb0["h2d/opt_states"] - r * 12 * n
    assert pb1.get("d2h/opt_states", 0) == pb0["d2h/opt_states"] - r * 12 * n


def test_warm_file_lane_changes_no_result(cuda_dev, tmp_path):
    # warm_files (default on) writes the activation / checkpoint extents once
    # and DMA-reads once into every file-read target before calibration: the
    # final states must equal the cold run's and the host tier's bit for bit
    # (ring and per-chunk host copies), every checkpoint must still round-trip
    # through the file, and the setup IO is reported, untimed
    sc = scenario(hardware='{"preset": "a100-12ssd", "cpu_mem": 1000000000}')
    base = {"compute_rate": RATE, "checksum_states": True, "seed": 9}
    st, host, _, err = execute(sc, dict(base, tier="host"))
    assert st == 0, (err, _failing(host))
    assert host["file_warmup_s"] == 0.0
    for ring in (0, 2):
        runs = {}
        for warm in (True, False):
            st, s, _, err = execute(sc, dict(base, tier="file", file_dir=str(tmp_path), host_ring=ring,
                                             warm_files=warm))
            assert st == 0, (err, _failing(s))
            assert s["all_invariants_pass"] and s["swap_mismatches"] == 0 and s["swap_checks"] == L
            assert s["checkpoint_location"] == "ssd"
            runs[warm] = s
        assert runs[True]["state_checksum"] == runs[False]["state_checksum"] == host["state_checksum"] != 0
        assert runs[True]["file_warmup_s"] > 0.0 and runs[False]["file_warmup_s"] == 0.0
        # the warm-up's requests are not the iteration's
        assert runs[True]["io_requests"]["fixed"] + runs[True]["io_requests"]["plain"] == \
            runs[False]["io_requests"]["fixed"] + runs[False]["io_requests"]["plain"]
        assert runs[True]["physical_bytes"] == runs[False]["physical_bytes"]
