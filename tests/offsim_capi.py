"""ctypes driver of the offsim C ABI (offsim_c.h), used to compare the
product library with the compiled reference (test infrastructure)."""
import ctypes as C
import hashlib
from pathlib import Path

PRESETS = ["13b-a100-b8", "13b-a100-b16", "13b-a100-b32", "13b-a100-b64", "13b-a100-b80",
           "13b-4090-b32", "175b-a100-b16", "175b-4090-b8"]
VARIANTS = ["serial", "pipelined", "overlapped"]

SCENARIO_DOCS = {
    "inline-gpt2": """{"schema_version": 1,
      "model": {"name": "gpt2-small-shape", "num_layers": 12, "num_heads": 12, "hidden_dim": 768,
                "batch_size": 8, "seq_len": 1024},
      "hardware": {"preset": "a100-12ssd"}, "variant": "overlapped", "planner": {"mode": "auto"},
      "seed": 7}""",
    "inline-gpt2-b128": """{"schema_version": 1,
      "model": {"name": "gpt2-small-shape", "num_layers": 12, "num_heads": 12, "hidden_dim": 768,
                "batch_size": 128, "seq_len": 1024},
      "hardware": "a100-12ssd"}""",
    "fixed-df": """{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 64},
      "hardware": {"preset": "a100-12ssd", "n_ssd": 6}, "variant": "pipelined",
      "planner": {"mode": "fixed_d_f", "d_f": 5e10}}""",
    "fixed-coef": """{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 32},
      "hardware": {"preset": "rtx4090-12ssd"}, "planner": {"mode": "fixed_coefficient",
      "coefficient": 0.3}}""",
    "13b-s2048-b32": """{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 32,
      "seq_len": 2048}, "hardware": "a100-12ssd"}""",
    "13b-s2048-b64": """{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 64,
      "seq_len": 2048}, "hardware": "a100-12ssd"}""",
    "low-cpu-mem": """{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": 16},
      "hardware": {"preset": "a100-12ssd", "cpu_mem": 200000000000}}""",
}

BAD_DOCS = {
    "bad-json": "{not json",
    "no-schema": '{"model": "gpt3-13b", "hardware": "a100-12ssd"}',
    "bad-schema": '{"schema_version": 2, "model": "gpt3-13b", "hardware": "a100-12ssd"}',
    "unknown-key": '{"schema_version": 1, "model": "gpt3-13b", "hardware": "a100-12ssd", "x": 1}',
    "unknown-model-key": '{"schema_version": 1, "model": {"preset": "gpt3-13b", "depth": 3}, "hardware": "a100-12ssd"}',
    "missing-hw-key": '{"schema_version": 1, "model": "gpt3-13b", "hardware": {"bw_gpu": 1}}',
    "bad-heads": '{"schema_version": 1, "model": {"num_layers": 2, "num_heads": 3, "hidden_dim": 64}, "hardware": "a100-12ssd"}',
    "bad-planner": '{"schema_version": 1, "model": "gpt3-13b", "hardware": "a100-12ssd", "planner": {"mode": "magic"}}',
    "bad-variant": '{"schema_version": 1, "model": "gpt3-13b", "hardware": "a100-12ssd", "variant": "fast"}',
    "bad-value": '{"schema_version": 1, "model": {"preset": "gpt3-13b", "batch_size": "x"}, "hardware": "a100-12ssd"}',
}


def load_offsim(path: Path) -> C.CDLL:
    lib = C.CDLL(str(path))
    P, S = C.c_void_p, C.c_int
    sigs = {
        "offsim_version": (C.c_char_p, []), "offsim_last_error": (C.c_char_p, []),
        "offsim_string_free": (None, [P]),
        "offsim_scenario_parse": (S, [C.c_char_p, C.POINTER(P)]),
        "offsim_scenario_from_preset": (S, [C.c_char_p, C.POINTER(P)]),
        "offsim_scenario_free": (None, [P]),
        "offsim_scenario_to_json": (S, [P, C.POINTER(P)]),
        "offsim_scenario_override": (S, [P, C.c_char_p, C.c_char_p]),
        "offsim_preset_names": (S, [C.POINTER(P)]),
        "offsim_plan": (S, [P, C.POINTER(P)]),
        "offsim_simulate": (S, [P, C.POINTER(P), C.POINTER(P)]),
        "offsim_sweep": (S, [P, C.c_char_p, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.POINTER(P)]),
        "offsim_capacity": (S, [P, C.POINTER(C.c_double), C.c_size_t, C.POINTER(P)]),
        "offsim_validate": (S, [P, C.POINTER(P)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


def _take(lib, p):
    if not p.value:
        return None
    s = C.cast(p, C.c_char_p).value.decode()
    lib.offsim_string_free(p)
    return s


def capi_outputs(lib, hashed=False, with_sweeps=True):
    """Every C-ABI output for a fixed set of inputs: {key: text or sha256}."""
    out = {}

    def put(key, text):
        out[key] = hashlib.sha256(text.encode()).hexdigest() if hashed and text is not None else text

    def scenario(kind, arg):
        h = C.c_void_p()
        fn = lib.offsim_scenario_from_preset if kind == "preset" else lib.offsim_scenario_parse
        st = fn(arg.encode(), C.byref(h))
        return st, h

    names = C.c_void_p()
    put("preset_names", f"{lib.offsim_preset_names(C.byref(names))}|{_take(lib, names)}")
    handles = [("preset:" + p, "preset", p) for p in PRESETS] + \
              [("doc:" + k, "doc", v) for k, v in SCENARIO_DOCS.items()]
    for key, kind, arg in handles:
        st, h = scenario(kind, arg)
        assert st == 0, (key, lib.offsim_last_error())
        j = C.c_void_p()
        put(key + "/to_json", f"{lib.offsim_scenario_to_json(h, C.byref(j))}|{_take(lib, j)}")
        variants = VARIANTS if kind == "preset" else [None]
        for v in variants:
            if v is not None:
                assert lib.offsim_scenario_override(h, b"variant", v.encode()) == 0
            tag = f"{key}/{v or 'doc'}"
            r = C.c_void_p()
            st = lib.offsim_plan(h, C.byref(r))
            put(tag + "/plan", f"{st}|{_take(lib, r)}|{lib.offsim_last_error().decode() if st else ''}")
            summ, tr = C.c_void_p(), C.c_void_p()
            st = lib.offsim_simulate(h, C.byref(summ), C.byref(tr))
            put(tag + "/simulate", f"{st}|{_take(lib, summ)}|{lib.offsim_last_error().decode() if st else ''}")
            put(tag + "/trace", _take(lib, tr))
        r = C.c_void_p()
        st = lib.offsim_validate(h, C.byref(r))
        put(key + "/validate", f"{st}|{_take(lib, r)}")
        lib.offsim_scenario_free(h)

    if with_sweeps:
        st, h = scenario("preset", "13b-a100-b32")
        vals = (C.c_double * 4)(8, 16, 32, 64)
        csv = C.c_void_p()
        put("sweep/batch", f"{lib.offsim_sweep(h, b'batch_size', vals, 4, 3, C.byref(csv))}|{_take(lib, csv)}")
        vals2 = (C.c_double * 4)(2, 4, 6, 12)
        put("sweep/n_ssd", f"{lib.offsim_sweep(h, b'n_ssd', vals2, 4, 1, C.byref(csv))}|{_take(lib, csv)}")
        vals3 = (C.c_double * 3)(0.0, 0.5, 1.0)
        put("sweep/coef", f"{lib.offsim_sweep(h, b'swap_coefficient', vals3, 3, 2, C.byref(csv))}|{_take(lib, csv)}")
        mem = (C.c_double * 6)(128, 256, 384, 512, 640, 768)
        put("capacity", f"{lib.offsim_capacity(h, mem, 6, C.byref(csv))}|{_take(lib, csv)}")
        st_bad = lib.offsim_sweep(h, b"depth", vals, 4, 1, C.byref(csv))
        put("sweep/bad-axis", f"{st_bad}|{lib.offsim_last_error().decode()}")
        for k, v in (("batch_size", "0"), ("planner", "2"), ("colour", "red"), ("variant", "x")):
            st = lib.offsim_scenario_override(h, k.encode(), v.encode())
            put(f"override/{k}={v}", f"{st}|{lib.offsim_last_error().decode()}")
        lib.offsim_scenario_free(h)
        # infeasible: 175B on the 4090 at batch 96 (reference CLI WILL_FAIL test)
        st, h = scenario("preset", "175b-4090-b8")
        assert lib.offsim_scenario_override(h, b"batch_size", b"96") == 0
        r = C.c_void_p()
        st = lib.offsim_plan(h, C.byref(r))
        put("infeasible/plan", f"{st}|{lib.offsim_last_error().decode()}|{r.value is None}")
        lib.offsim_scenario_free(h)

    for k, doc in BAD_DOCS.items():
        h = C.c_void_p()
        st = lib.offsim_scenario_parse(doc.encode(), C.byref(h))
        put("bad/" + k, f"{st}|{lib.offsim_last_error().decode()}|{h.value is None}")
    h = C.c_void_p()
    st = lib.offsim_scenario_from_preset(b"nope", C.byref(h))
    put("bad/preset", f"{st}|{lib.offsim_last_error().decode()}")
    st = lib.offsim_plan(None, C.byref(h))
    put("bad/null", f"{st}|{lib.offsim_last_error().decode()}")
    return out
