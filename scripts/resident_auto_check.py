"""resident_groups auto on a 12-block 65B-shaped slice (states 116 GB): how many groups the
executor keeps in HBM, and the iteration with / without them. usage: python scripts/resident_auto_check.py"""
import sys, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import exec_api as X
sc = X.scenario(layers=12, heads=64, hidden=8192, batch=4, seq=1024, name="65b-shape-12-blocks")
for opts in ({"tier": "host", "compute_rate": 1.4e15}, {"tier": "host", "compute_rate": 1.4e15, "resident_groups": "auto"}):
    st, s, _, err = X.execute(sc, opts)
    print(json.dumps({"opts": opts, "status": st, "err": err[:200], "resident_groups": s and s.get("resident_groups"),
                      "executed_s": s and s["executed"]["makespan_s"], "predicted_s": s and s["predicted"]["makespan_s"],
                      "invariants": s and s["all_invariants_pass"],
                      "h2d_states_gb": s and s["physical_bytes"].get("h2d/opt_states", 0) / 1e9}))
