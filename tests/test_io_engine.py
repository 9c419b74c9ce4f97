"""CPU: the file-tier IO engine (io_uring on raw syscalls, O_DIRECT, with a
pread/pwrite fallback) round-trips data bit-exactly, including a tail that
is not a multiple of the request size (build/io_engine_test, linked against
the product's csrc/core/io_engine.cpp)."""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parents[1] / "build" / "io_engine_test"


@pytest.mark.parametrize("mib,depth", [(8, 32), (3, 1), (17, 4)])
def test_io_engine_round_trip(tmp_path, mib, depth):
    if not EXE.exists():
        pytest.skip("build/io_engine_test not built")
    r = subprocess.run([str(EXE), str(tmp_path), str(mib), str(depth)], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    engine, status = r.stdout.split()[:2]
    assert status == "OK"
    assert engine in ("io_uring", "pread/pwrite")


@pytest.mark.parametrize("depth", [1, 8])
def test_io_engine_reports_injected_faults(tmp_path, depth):
    """A write through a read-only fd and a read past EOF are reported as
    errors (never a crash or silent short data) — the executor turns them
    into OFFSIM_ERR_INFEASIBLE / FY_ERR_DEVICE."""
    if not EXE.exists():
        pytest.skip("build/io_engine_test not built")
    r = subprocess.run([str(EXE), str(tmp_path), "fault", str(depth)], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAULTS-REPORTED" in r.stdout


@pytest.mark.parametrize("mib,depth", [(8, 32), (3, 1), (17, 4)])
def test_io_engine_registered_buffers(tmp_path, mib, depth):
    """Registered (fixed) buffers: requests inside a registered buffer go out
    as READ_FIXED / WRITE_FIXED, a request straddling two registrations as a
    plain op (odd sizes split the read buffer mid-request), data bit-exact."""
    if not EXE.exists():
        pytest.skip("build/io_engine_test not built")
    r = subprocess.run([str(EXE), str(tmp_path), str(mib), str(depth), "fixed"], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    f = r.stdout.split()
    assert f[1] == "OK"
    kv = dict(x.split("=") for x in f[4:])
    if f[0] != "io_uring" or int(kv["registered"]) == 0:
        pytest.skip(f"registration unavailable here ({f[0]}, registered={kv['registered']})")
    assert int(kv["registered"]) == 2 * (mib << 20)
    straddle = mib % 2  # the read buffer's halves meet mid-request for odd MiB
    assert int(kv["plain"]) == straddle
    assert int(kv["fixed"]) == 2 * mib - straddle


@pytest.mark.parametrize("fixed", [False, True])
@pytest.mark.parametrize("count,mib", [(1, 3), (2, 7), (3, 7), (4, 13)])
def test_io_engine_striped_over_devices(tmp_path, count, mib, fixed):
    """RAID-0 striping over `count` files (the reference's n_ssd devices,
    hardware.cpp:39-42): a region at an offset that is not unit-aligned
    round-trips bit-exactly and every device file holds exactly the bytes
    the mapping assigns it."""
    if not EXE.exists():
        pytest.skip("build/io_engine_test not built")
    args = [str(EXE), str(tmp_path), "stripe", str(count), str(mib)] + (["fixed"] if fixed else [])
    r = subprocess.run(args, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    f = r.stdout.split()
    assert f[1:3] == ["STRIPE-OK", str(count)]
    kv = dict(x.split("=") for x in f[3:])
    if f[0] == "io_uring" and fixed and int(kv["fixed"]) > 0:
        assert int(kv["plain"]) == 0  # every striped request lies inside a registered buffer
    elif f[0] == "io_uring" and not fixed:
        assert int(kv["fixed"]) == 0
