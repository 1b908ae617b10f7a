"""tools/kronbench: the reference bench CLI (proj/tools/bench_main.cpp) on the
B200 library -- flag validation here (no GPU needed), verified runs and the
CSV schema on the GPU (-m gpu)."""
import csv
import io
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "kronbench", "kronbench")

needs_exe = pytest.mark.skipif(not os.path.exists(EXE), reason="kronbench not built (make kronbench)")


def run(*args, timeout=600):
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=timeout)


@needs_exe
@pytest.mark.parametrize("args, msg", [(["--sizes", "3..1"], "bad --sizes value '3..1'"),
                                       (["--sizes", "0"], "bad --sizes value"),
                                       (["--precision", "quad"], "--precision"),
                                       (["--dims", "4d"], "--dims"),
                                       (["--bogus"], "unknown option")])
def test_flag_errors(args, msg):
    r = run(*args)
    assert r.returncode == 1 and msg in r.stderr, r.stderr


@needs_exe
def test_help():
    r = run("--help")
    assert r.returncode == 0 and "--sizes" in r.stderr


@needs_exe
@pytest.mark.gpu
def test_verify_only_all_sizes():
    r = run("--verify-only", "--batch", "300", "--sizes", "1..16", "--resident")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if "verified" in l]
    assert len(lines) == 16 * 4


@needs_exe
@pytest.mark.gpu
@pytest.mark.parametrize("resident", [False, True])
def test_csv_schema(resident):
    args = ["--format", "csv", "--sizes", "10,16", "--batch", "2000", "--reps", "3", "--beta", "0.5", "--b200-columns"]
    r = run(*args, *(["--resident"] if resident else []))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert list(rows[0].keys())[:7] == ["size", "precision", "dims", "batch", "seconds", "gflops", "verified"]
    assert len(rows) == 8 and all(x["verified"] == "true" and float(x["gflops"]) > 0 for x in rows)
    assert all(x["mode"] == ("resident" if resident else "host") for x in rows)


@needs_exe
@pytest.mark.gpu
def test_csv_reference_schema_by_default():
    r = run("--format", "csv", "--sizes", "2,3", "--batch", "100", "--reps", "1")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "size,precision,dims,batch,seconds,gflops,verified"  # bench_support.cpp:346-352
    assert len(lines) == 9 and all(len(l.split(",")) == 7 for l in lines)
