"""CPU: the product library loads without a GPU and exports every function
declared in include/**/*.h (the drop-in boundary); pure-host entry points
behave (no CUDA compute is called here)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADERS = sorted((ROOT / "include").rglob("*.h"))
DECL = re.compile(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b((?:offsim|fy)_[a-z0-9_]+)\s*\(", re.M)


def declared():
    names = set()
    for h in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in DECL.finditer(text):
            if "typedef" in text[max(0, m.start() - 40):m.start() + 1].split("\n")[-1]:
                continue
            names.add(m.group(1))
    return sorted(names)


def test_headers_found():
    assert any(h.name == "fy_adam.h" for h in HEADERS)
    assert len(declared()) >= 10


@pytest.mark.parametrize("name", declared())
def test_symbol_exported(name):
    from paper_2403_06504_b200._lib import LIB
    assert hasattr(LIB, name), f"{name} declared in include/ but not exported"


def test_shard_range_partitions():
    from paper_2403_06504_b200 import optim as F
    for n in (1, 7, 8, 4099, 314572800, 7077888):
        for world in (1, 2, 3, 4, 8):
            covered = 0
            prev_end = 0
            for r in range(world):
                off, cnt = F.shard_range(n, world, r, 8)
                assert off == prev_end
                if r < world - 1 and cnt > 0 and off + cnt < n:
                    assert cnt % 8 == 0 and off % 8 == 0
                prev_end = off + cnt
                covered += cnt
            assert covered == n


def test_errors_are_status_codes():
    from paper_2403_06504_b200._lib import LIB, FY_ERR_CONFIG
    off, cnt = C.c_uint64(), C.c_uint64()
    assert LIB.fy_shard_range(10, 0, 0, 8, C.byref(off), C.byref(cnt)) == FY_ERR_CONFIG
    assert b"rank" in LIB.fy_last_error()
    assert LIB.fy_adamw_chunk(None, None) == FY_ERR_CONFIG
    assert LIB.fy_last_error() == b"null argument"
    assert LIB.fy_version().startswith(b"0.")


def test_argument_validation_without_gpu():
    """Every fy_* entry point validates its arguments before touching the
    device, with the reference C ABI's conventions (status codes, thread-local
    last error) — so these run on a CPU-only machine."""
    from paper_2403_06504_b200._lib import (LIB, AdamwArgs, AdamHparams, FY_ERR_CONFIG,
                                            PipelineConfig)
    a = AdamwArgs()
    a.n = 16
    a.master = a.exp_avg = a.exp_avg_sq = a.grad = 0x1000
    a.hp = AdamHparams(1e-4, 0.9, 0.95, 1e-8, 0.1, 0, 1, 1, 1.0)  # step 0
    assert LIB.fy_adamw_chunk(C.byref(a), None) == FY_ERR_CONFIG
    assert b"step" in LIB.fy_last_error()
    a.hp.step = 10
    a.grad_dtype = 7
    assert LIB.fy_adamw_chunk(C.byref(a), None) == FY_ERR_CONFIG
    assert b"grad_dtype" in LIB.fy_last_error()
    a.grad_dtype = 0
    a.grad_sq_sum = 0x2000  # without workspace
    assert LIB.fy_adamw_chunk(C.byref(a), None) == FY_ERR_CONFIG
    assert b"workspace" in LIB.fy_last_error()
    dst = (C.c_void_p * 9)(*([0x3000] * 9))
    a.grad_sq_sum = None
    a.param_out = 0x4000
    assert LIB.fy_adamw_chunk_gather(C.byref(a), dst, 9, None) == FY_ERR_CONFIG
    assert b"8" in LIB.fy_last_error()
    a.param_out = None
    assert LIB.fy_adamw_chunk_gather(C.byref(a), dst, 2, None) == FY_ERR_CONFIG
    assert b"param_out" in LIB.fy_last_error()
    assert LIB.fy_adamw_tune(2, 3, 0) == FY_ERR_CONFIG
    assert LIB.fy_adamw_tune(0, 3, 0) == FY_ERR_CONFIG
    assert LIB.fy_adamw_tune(1, 2, 0) == FY_ERR_CONFIG  # 2 stages: sweep build only
    assert LIB.fy_adamw_tune(1, 8, 0) == FY_ERR_CONFIG
    assert LIB.fy_adamw_tune(1, 3, 4) == FY_ERR_CONFIG  # 4 consumer warps: sweep build only
    assert not hasattr(LIB, "fy_adamw_tune_bulk"), "sweep-only variants must not ship in the product"
    h = C.c_void_p()
    cfg = PipelineConfig(0, 1024, 1, 0, 0, 0, 1, 0, 0)
    assert LIB.fy_pipeline_create(C.byref(cfg), C.byref(h)) == FY_ERR_CONFIG
    assert b"slots" in LIB.fy_last_error()
    cfg = PipelineConfig(0, 0, 3, 0, 0, 0, 1, 0, 0)
    assert LIB.fy_pipeline_create(C.byref(cfg), C.byref(h)) == FY_ERR_CONFIG
    cfg = PipelineConfig(0, 1024, 3, 0, 2, 0, 1, 0, 0)  # fp32 params
    assert LIB.fy_pipeline_create(C.byref(cfg), C.byref(h)) == FY_ERR_CONFIG
    assert LIB.fy_pipeline_step(None, None, 0, None, 0) == FY_ERR_CONFIG
    assert LIB.fy_pipeline_wait(None, None, None) == FY_ERR_CONFIG
    assert LIB.fy_host_alloc(16, None) == FY_ERR_CONFIG
    out = C.c_void_p()
    assert LIB.fy_host_alloc_on(16, -3, C.byref(out)) == FY_ERR_CONFIG
    assert LIB.fy_device_numa_node(0, None) == FY_ERR_CONFIG
    assert LIB.fy_host_numa_node(None, None) == FY_ERR_CONFIG
    assert LIB.fy_clip_coef(None, None, 1.0, None, None, None) == FY_ERR_CONFIG
    assert LIB.fy_clip_coef(0x1000, None, -1.0, 0x2000, None, None) == FY_ERR_CONFIG
    assert b"max_norm" in LIB.fy_last_error()
    assert LIB.fy_adamw_chunks(None, 3, None) == FY_ERR_CONFIG
    assert LIB.fy_swapper_create(None, None) == FY_ERR_CONFIG
    h = C.c_uint64()
    assert LIB.fy_swap_out(None, None, 16, 0, None, None, C.byref(h)) == FY_ERR_CONFIG
    assert LIB.fy_swap_in(None, 1, None, None, None) == FY_ERR_CONFIG
    assert LIB.fy_swap_release(None, 1) == FY_ERR_CONFIG
    assert LIB.fy_swapper_sync(None) == FY_ERR_CONFIG
    assert LIB.fy_ipc_alloc(0, None, None) == FY_ERR_CONFIG
    assert LIB.fy_ipc_open(None, None) == FY_ERR_CONFIG
    assert LIB.fy_ipc_close(None) == FY_ERR_CONFIG


def test_graph_execute_rejects_bad_input_without_gpu():
    from paper_2403_06504_b200._lib import LIB, Chunk
    LIB.fy_graph_execute.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(Chunk), C.c_uint32,
                                     C.POINTER(C.c_void_p)]
    LIB.offsim_last_error.restype = C.c_char_p
    out = C.c_void_p()
    assert LIB.fy_graph_execute(b"{bad", None, None, 0, C.byref(out)) == 2
    assert LIB.fy_graph_execute(None, None, None, 0, C.byref(out)) == 2
    sc = (b'{"schema_version": 1, "model": {"num_layers": 2, "num_heads": 4, "hidden_dim": 64},'
          b' "hardware": "a100-12ssd"}')
    arr = (Chunk * 2)()
    arr[0].n = arr[1].n = 12 * 64 * 64 + 1  # wrong chunk size
    assert LIB.fy_graph_execute(sc, None, arr, 2, C.byref(out)) == 2
    assert b"12*h^2" in LIB.offsim_last_error()
    assert LIB.fy_graph_execute(sc, b'{"tier": "disk"}', None, 0, C.byref(out)) == 2
    assert not out.value


def test_c_consumer_compiles_links_and_runs(tmp_path):
    """A plain C11 program (no C++, no CUDA headers) includes both public C
    headers, links liboffsim.so.0 and calls into it — what a cgo / JNI /
    N-API / ctypes binding does."""
    import shutil
    import subprocess
    from pathlib import Path
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_2403_06504_b200" / "lib"
    src = tmp_path / "consumer.c"
    src.write_text(r'''
#include "fuyou/fy_adam.h"
#include "offsim/offsim_c.h"
#include <stdio.h>
#include <string.h>
int main(void) {
    char* report = NULL;
    offsim_scenario* s = NULL;
    if (offsim_scenario_from_preset("13b-a100-b32", &s) != OFFSIM_OK) return 2;
    if (offsim_plan(s, &report) != OFFSIM_OK || !report || !strstr(report, "swap_coefficient")) return 3;
    offsim_string_free(report);
    offsim_scenario_free(s);
    uint64_t off = 0, cnt = 0;
    if (fy_shard_range(1000, 3, 1, 8, &off, &cnt) != FY_OK || off == 0 || cnt == 0) return 4;
    if (fy_adamw_chunk(NULL, NULL) != FY_ERR_CONFIG || fy_last_error() == NULL) return 5;
    printf("%s %s\n", offsim_version(), fy_version());
    return 0;
}
''')
    exe = tmp_path / "consumer"
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", f"-I{root / 'include'}", str(src),
                        f"-L{lib}", "-l:liboffsim.so.0", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
