"""ctypes helpers for the executor entry points (offsim_execute,
fy_graph_execute) of the product library."""
import ctypes as C
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PRODUCT = ROOT / "paper_2403_06504_b200" / "lib" / "liboffsim.so.0"


def lib():
    from paper_2403_06504_b200._lib import LIB, Chunk
    L = LIB
    P = C.c_void_p
    L.offsim_scenario_parse.argtypes = [C.c_char_p, C.POINTER(P)]
    L.offsim_scenario_parse.restype = C.c_int
    L.offsim_scenario_free.argtypes = [P]
    L.offsim_execute.argtypes = [P, C.c_char_p, C.POINTER(P), C.POINTER(P)]
    L.offsim_execute.restype = C.c_int
    L.offsim_string_free.argtypes = [P]
    L.offsim_last_error.restype = C.c_char_p
    L.fy_graph_execute.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(Chunk), C.c_uint32, C.POINTER(P)]
    L.fy_graph_execute.restype = C.c_int
    return L


def _take(L, p):
    if not p.value:
        return None
    s = C.cast(p, C.c_char_p).value.decode()
    L.offsim_string_free(p)
    return s


def execute(scenario: str, opts: dict, want_trace=False):
    L = lib()
    h = C.c_void_p()
    st = L.offsim_scenario_parse(scenario.encode(), C.byref(h))
    assert st == 0, L.offsim_last_error()
    summ, tr = C.c_void_p(), C.c_void_p()
    st = L.offsim_execute(h, json.dumps(opts).encode(), C.byref(summ),
                          C.byref(tr) if want_trace else None)
    L.offsim_scenario_free(h)
    err = L.offsim_last_error().decode() if st else ""
    s = _take(L, summ)
    return st, (json.loads(s) if s else None), (_take(L, tr) if want_trace else None), err


def graph_execute(scenario: str, opts: dict, chunks):
    from paper_2403_06504_b200._lib import Chunk
    L = lib()
    arr = (Chunk * len(chunks))()
    for i, c in enumerate(chunks):
        arr[i] = Chunk(c["n"], c["h_states"], c["grad"], c["h_param"], None, None, 0, None, 0)
    summ = C.c_void_p()
    st = L.fy_graph_execute(scenario.encode(), json.dumps(opts).encode(), arr, len(chunks),
                            C.byref(summ))
    err = L.offsim_last_error().decode() if st else ""
    s = _take(L, summ)
    return st, (json.loads(s) if s else None), err


def scenario(layers=12, heads=12, hidden=768, batch=8, seq=1024, hardware='"a100-12ssd"',
             variant="overlapped", name="gpt2-small-shape"):
    return json.dumps({"schema_version": 1,
                       "model": {"name": name, "num_layers": layers, "num_heads": heads,
                                 "hidden_dim": hidden, "batch_size": batch, "seq_len": seq},
                       "hardware": json.loads(hardware), "variant": variant})
