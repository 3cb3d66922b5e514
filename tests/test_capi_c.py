"""The drop-in proof in C (tests/capi/capi_c_test.c): a plain-C caller compiled against
include/strassen.h and linked to libstrassen_b200.so, porting the reference's
test_capi.cpp and its bench's run_once / rank-b / verification (bench_lib.cpp:56-71,
208-269).  Without a device only the checks that make no compute call run."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "capi_c_test")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "capi")], check=True)


def test_c_caller_compiles_and_links_against_the_header():
    _build()
    r = subprocess.run([EXE, "--no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


@pytest.mark.gpu
def test_c_caller_full_suite_on_device(cuda):
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [ln.split(",") for ln in r.stdout.splitlines() if ln[:1].isdigit()]
    assert len(rows) == 21  # 3 shapes x the reference's 7 configurations
    for row in rows:
        egf_modeled, rel_err = float(row[9]), float(row[10])
        assert egf_modeled > 0.0
        assert rel_err < 1e-11
    print(r.stdout.splitlines()[-1])
