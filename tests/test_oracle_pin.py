"""Pin the oracle, then run the reference's own suites against the product.

1. oracle/_ref: the unmodified reference compiled in place; its own doctest
   suites and the 10 acceptance criteria must pass (this is what makes it a
   trustworthy oracle).
2. drop-in: the same suites compiled against THIS repo's hot path
   (kv_manager/scheduler/sim_engine/cost_model replaced), must also pass.
3. differential fuzz: product vs reference in one binary, bit-identical.

Needs /root/reference to build; on a box without it the prebuilt binaries in
oracle/_ref and tests/native/_build are used when present, else skipped.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref")
NATIVE = os.path.join(ROOT, "tests", "native")
DROPIN = os.path.join(NATIVE, "_build", "dropin")
SUITES = ["test_cost_model", "test_workload", "test_kv_manager", "test_placement", "test_scheduler",
          "test_sim_engine", "test_metrics", "test_cli", "acceptance"]
HAVE_REF = os.path.isdir("/root/reference/proj")


def _ensure(target_dir, make_dir, target):
    path = os.path.join(target_dir, target)
    if HAVE_REF and shutil.which("make"):
        subprocess.run(["make", "-s", "-j8", "-C", make_dir], check=True, capture_output=True)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built and /root/reference absent")
    return path


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_oracle(suite):
    exe = _ensure(REF_BIN, os.path.join(ROOT, "oracle"), suite)
    r = subprocess.run([exe], cwd=REF_BIN, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed | checks" in r.stdout


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_product(suite):
    exe = _ensure(DROPIN, NATIVE, suite)
    r = subprocess.run([exe], cwd=DROPIN, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    if suite == "acceptance":
        assert r.stdout.count("PASS") == 10, r.stdout


def test_acceptance_outputs_identical():
    """Every acceptance verdict line (throughputs, gaps, counts) is the same
    with the product hot path as with the reference."""
    a = _ensure(REF_BIN, os.path.join(ROOT, "oracle"), "acceptance")
    b = _ensure(DROPIN, NATIVE, "acceptance")
    ra = subprocess.run([a], cwd=REF_BIN, capture_output=True, text=True, timeout=600).stdout
    rb = subprocess.run([b], cwd=DROPIN, capture_output=True, text=True, timeout=600).stdout
    strip = lambda s: [l.split(", 0.")[0].rsplit(" s wall", 1)[0] for l in s.splitlines() if l.startswith("ACCEPT")]
    assert strip(ra) == strip(rb)


@pytest.mark.parametrize("mode,count", [("pool", 3000), ("phys", 3000), ("sim", 60)])
def test_differential_fuzz(mode, count):
    exe = _ensure(os.path.join(NATIVE, "_build"), NATIVE, "diff_fuzz")
    r = subprocess.run([exe, mode, "7", str(count)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout
