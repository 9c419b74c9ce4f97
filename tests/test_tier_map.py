"""CPU: the B200 tier map (map_graph_for_b200) through offsim_execute's dry
run — inserted optimizer hops, bytes that stay in HBM / pinned DRAM, the
slot-reuse edges, and the UNCHANGED trace invariants on the mapped graph."""
import pytest

from exec_api import execute, scenario

C1 = scenario()                                       # GPT-2-small shape, b=8
C1_SSD = scenario(hardware='{"preset": "a100-12ssd", "cpu_mem": 1000000000}')
C2 = scenario(40, 40, 5120, 32, 1024, name="gpt3-13b")
N1, L1 = 12 * 768 * 768, 12
N2, L2 = 12 * 5120 * 5120, 40


@pytest.mark.parametrize("sc,N,L", [(C1, N1, L1), (C2, N2, L2)])
def test_host_tier_overlapped(sc, N, L):
    st, s, _, err = execute(sc, {"dry_run": True, "tier": "host"})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    assert s["task_count"] == s["reference_task_count"] + 3 * L
    assert len(s["inserted_tasks"]) == 3 * L
    mb = s["mapped_bytes"]
    assert all(v == 0 for k, v in mb.items() if k.startswith("link_ssd/"))
    assert mb.get("link_g2c/grads", 0) == 0          # grads stay in HBM
    assert mb["link_c2g/opt_states"] == 12 * N * L     # states in (12 B/param)
    assert mb["link_g2c/opt_states"] == 12 * N * L     # states out
    ref = s["reference_bytes"]
    assert mb["link_g2c/params"] == 2 * N * L          # bf16 params out
    assert ref["link_ssd/opt_states"] == 24 * N * L    # reference: 12N read + 12N write


def test_file_tier_keeps_reference_ssd_bytes():
    st, s, _, err = execute(C1_SSD, {"dry_run": True, "tier": "file"})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    ref, mb = s["reference_bytes"], s["mapped_bytes"]
    for k, v in ref.items():
        if k.startswith("link_ssd/") and k != "link_ssd/grads":
            assert mb[k] == v, k
    assert any(k == "link_ssd/activations" for k in mb)  # checkpoints go to the file tier


@pytest.mark.parametrize("variant", ["serial", "pipelined"])
def test_non_overlapped_variants(variant):
    sc = scenario(variant=variant)
    st, s, _, err = execute(sc, {"dry_run": True, "tier": "host"})
    assert st == 2 and "tier=file" in err
    st, s, _, err = execute(sc, {"dry_run": True, "tier": "file"})
    assert st == 0, err
    names = {e["name"]: e["pass"] for e in s["invariants"]}
    assert names["gradient-ssd-roundtrip"]
    assert s["all_invariants_pass"], s["invariants"]
    assert len(s["inserted_tasks"]) == 4 * L1  # + grad_h2d per group


def test_slot_edges_and_bad_options():
    st, s, _, err = execute(C1, {"dry_run": True, "state_slots": 2})
    assert st == 0 and s["all_invariants_pass"]
    st, _, _, err = execute(C1, {"dry_run": True, "state_slots": 1})
    assert st == 2 and "state_slots" in err
    st, _, _, err = execute(C1, {"dry_run": True, "colour": "red"})
    assert st == 2 and "colour" in err
    st, _, _, err = execute(C1, {"dry_run": True, "tier": "tape"})
    assert st == 2


def test_swap_only_subgraph_c5():
    # BASELINE config 5 at b=32 (coefficient 1, all 160 layers swapped):
    # the swap path of 2 blocks = 2 checkpoints + 8 activations, out and back
    sc = scenario(40, 40, 5120, 32, 2048, name="gpt3-13b")
    st, s, _, err = execute(sc, {"dry_run": True, "swap_only": True, "max_blocks": 2})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    assert s["task_count"] == 2 * (2 + 8)  # g2c + c2g per unit (cpu placement)
    per_block = 32 * 2048 * 5120 * 10
    assert s["mapped_bytes"]["link_g2c/activations"] == 2 * per_block
    assert s["mapped_bytes"]["link_c2g/activations"] == 2 * per_block
    st, s, _, err = execute(sc, {"dry_run": True, "swap_only": True, "max_blocks": 2,
                                 "placement": "ssd", "tier": "file"})
    assert st == 0, err
    assert s["task_count"] == 4 * (2 + 8)  # + c2s and s2c legs
    assert s["mapped_bytes"]["link_ssd/activations"] == 2 * 2 * per_block


@pytest.mark.parametrize("ring", [1, 2, 4])
def test_host_ring_edges_keep_invariants(ring):
    # bounded staging rings on the file tier with checkpoints on SSD: the
    # ring-reuse edges must keep the graph a DAG the unchanged checks accept
    st, s, _, err = execute(C1_SSD, {"dry_run": True, "tier": "file", "host_ring": ring})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    base = execute(C1_SSD, {"dry_run": True, "tier": "file"})[1]
    # the same tasks and bytes; only extra ordering
    assert s["task_count"] == base["task_count"]
    assert s["mapped_bytes"] == base["mapped_bytes"]
    # (no makespan monotonicity check: FIFO list scheduling has Graham
    # anomalies — an extra edge can shorten the DES makespan)


def test_host_ring_auto_follows_reference_windows():
    # "auto": ring depths come from the windows build_schedule sized
    # (task_graph.cpp:145-224) — weights = the CPU stage window in blocks,
    # activations = the offload window x units per block, states/params =
    # the device staging slots — clamped to [2, uses]
    st, s, _, err = execute(C1_SSD, {"dry_run": True, "tier": "file", "host_ring": "auto"})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    w, r = s["windows"], s["host_ring"]
    assert r["states"] == r["params"] == 3
    assert r["weights"] == min(max((w["cpu_stage_window_layers"] + 3) // 4, 2), 2 * 4 * 12)
    assert 2 <= r["acts"] <= 2 * (12 * 4 + 12)
    assert r["acts"] >= min(w["offload_window_blocks"], 24)
    st, s4, _, _ = execute(C1_SSD, {"dry_run": True, "tier": "file", "host_ring": 4})
    assert s4["host_ring"] == {"states": 4, "params": 4, "weights": 4, "acts": 4}
    st, s0, _, _ = execute(C1_SSD, {"dry_run": True, "tier": "host", "host_ring": "auto"})
    assert s0["host_ring"] == {"states": 0, "params": 0, "weights": 0, "acts": 0}
    st, _, _, err = execute(C1_SSD, {"dry_run": True, "tier": "file", "host_ring": "many"})
    assert st == 2 and "auto" in err


@pytest.mark.parametrize("tier,R", [("host", 3), ("file", 2), ("host", "all")])
def test_resident_groups_move_no_state_bytes(tier, R):
    """resident_groups: optimizer groups g0..g(R-1) keep master/m/v in HBM —
    their state hops (and, file tier, state file IO) move 0 B, the GPU pool
    books their 12N B from the start, and the unchanged invariants still
    hold on the mapped graph's DES."""
    sc = C1_SSD if tier == "file" else C1
    st, base, _, err = execute(sc, {"dry_run": True, "tier": tier})
    assert st == 0, err
    st, s, _, err = execute(sc, {"dry_run": True, "tier": tier, "resident_groups": R})
    assert st == 0, err
    assert s["all_invariants_pass"], s["invariants"]
    r = L1 if R == "all" else R
    mb, b0 = s["mapped_bytes"], base["mapped_bytes"]
    assert mb.get("link_c2g/opt_states", 0) == b0["link_c2g/opt_states"] - 12 * N1 * r
    assert mb.get("link_g2c/opt_states", 0) == b0["link_g2c/opt_states"] - 12 * N1 * r
    assert mb["link_g2c/params"] == b0["link_g2c/params"]     # params still go to host
    if tier == "file":
        assert mb["link_ssd/opt_states"] == b0["link_ssd/opt_states"] - 24 * N1 * r


def test_resident_groups_rejects_bad_value():
    st, _, _, err = execute(C1, {"dry_run": True, "resident_groups": "some"})
    assert st == 2 and "resident_groups" in err


def test_file_dir_list_for_striping():
    """file_dir may list one directory per SSD (tier files striped over
    them); an empty list or a non-string entry is a config error."""
    st, s, _, err = execute(C1, {"dry_run": True, "tier": "file", "file_dir": ["/tmp/a", "/tmp/b"]})
    assert st == 0 and s["all_invariants_pass"], err
    st, _, _, err = execute(C1, {"dry_run": True, "tier": "file", "file_dir": []})
    assert st == 2 and "file_dir" in err
    st, _, _, err = execute(C1, {"dry_run": True, "tier": "file", "file_dir": ["/tmp/a", 3]})
    assert st == 2
    st, _, _, err = execute(C1, {"dry_run": True, "tier": "file", "file_dir": ["/tmp/a", "/tmp/a"]})
    assert st == 2 and "distinct" in err


def test_io_depth_option():
    """io_depth = io_uring requests in flight per tier device (1..1024)."""
    st, s, _, err = execute(C1, {"dry_run": True, "tier": "file", "io_depth": 64})
    assert st == 0, err
    for bad in (0, 2000):
        st, _, _, err = execute(C1, {"dry_run": True, "tier": "file", "io_depth": bad})
        assert st == 2 and "io_depth" in err


def test_warm_files_option():
    """warm_files (default true) is a bool exec option; a non-bool is a config error."""
    for v in (True, False):
        st, s, _, err = execute(C1, {"dry_run": True, "tier": "file", "warm_files": v})
        assert st == 0, err
    st, _, _, err = execute(C1, {"dry_run": True, "tier": "file", "warm_files": "yes"})
    assert st == 2


def test_ssd_link_overlap_reported():
    """The file lane's planned overlap with the link lanes (the weight of its
    copy-engine-loaded replay): in [0, 1]; > 0 when states stream through
    files and pinned memory at once; 0 on the host tier (no file lane)."""
    st, s, _, err = execute(C1, {"dry_run": True, "tier": "file"})
    assert st == 0, err
    f = s["link_overlap"]["ssd_link"]
    assert 0.0 < f <= 1.0, f
    st, s, _, err = execute(C1, {"dry_run": True, "tier": "host"})
    assert st == 0, err
    assert s["link_overlap"]["ssd_link"] == 0.0


def _dry_trace(sc, opts):
    import json
    st, s, tr, err = execute(sc, {"dry_run": True, **opts}, want_trace=True)
    assert st == 0, err
    d = json.loads(tr)
    lanes = {e["tid"]: e["args"]["name"] for e in d["traceEvents"] if e.get("ph") == "M"
             and e["name"] == "thread_name"}
    ev = [(lanes[e["tid"]], e["name"], e["ts"], e["dur"]) for e in d["traceEvents"] if e.get("ph") == "X"]
    return s, ev


@pytest.mark.parametrize("sc,opts", [(C1, {"tier": "host"}), (C1, {"tier": "host", "resident_groups": "all"}),
                                     (C2, {"tier": "host"})])
def test_analytic_model_is_per_phase_busiest_lane(sc, opts):
    """analytic_iteration (the reference cost model's structure on the mapped
    graph, cost_model.cpp:26-90): t_f / t_bo = the busiest lane's summed
    task durations over the forward tasks / the backward + optimizer tasks;
    recomputed here from the DES trace's own durations."""
    from collections import defaultdict
    s, ev = _dry_trace(sc, opts)
    phase = {"fwd": defaultdict(float), "rest": defaultdict(float)}
    for lane, name, ts, dur in ev:
        phase["fwd" if name.startswith("fwd ") else "rest"][lane] += dur * 1e-6
    a = s["analytic"]
    assert a["t_f_s"] == pytest.approx(max(phase["fwd"].values()), rel=1e-6)
    assert a["t_bo_s"] == pytest.approx(max(phase["rest"].values()), rel=1e-6)
    assert a["t_iter_s"] == pytest.approx(a["t_f_s"] + a["t_bo_s"], rel=1e-12)
    assert a["t_iter_s"] <= s["planned"]["makespan_s"] * 2.0


@pytest.mark.parametrize("sc,opts", [(C1, {"tier": "host"}), (C1, {"tier": "host", "resident_groups": "all"}),
                                     (C2, {"tier": "host"})])
def test_link_overlap_matches_trace(sc, opts):
    """link_overlap: the share of each link lane's busy time during which the
    other direction is busy (the weight of the duplex-loaded replay in the
    effective link rate), recomputed from the DES trace's intervals."""
    s, ev = _dry_trace(sc, opts)
    up = sorted((ts, ts + dur) for lane, _, ts, dur in ev if lane == "CPU to GPU" and dur > 0)
    down = sorted((ts, ts + dur) for lane, _, ts, dur in ev if lane == "GPU to CPU" and dur > 0)
    both, i, j = 0.0, 0, 0
    while i < len(up) and j < len(down):
        lo, hi = max(up[i][0], down[j][0]), min(up[i][1], down[j][1])
        both += max(0.0, hi - lo)
        if up[i][1] < down[j][1]:
            i += 1
        else:
            j += 1
    lo = s["link_overlap"]
    assert lo["c2g"] == pytest.approx(both / sum(b - a for a, b in up), abs=1e-6)
    assert lo["g2c"] == pytest.approx(both / sum(b - a for a, b in down), abs=1e-6)
    assert 0.0 <= lo["c2g"] <= 1.0 and 0.0 <= lo["g2c"] <= 1.0
