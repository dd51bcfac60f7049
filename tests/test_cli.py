"""`qsv run` report driver: flags, RunReport JSON/CSV with
identical values, device-side verification; fails loudly without a GPU (no CPU fallback)."""
import csv
import io
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
QSV = os.path.join(ROOT, "paper_2509_04955_b200", "lib", "qsv")


def run(*args):
    return subprocess.run([QSV, *args], capture_output=True, text=True, timeout=600)


def test_cli_usage_errors():
    assert run().returncode == 2
    r = run("run", "--gen", "qft:8", "--fusion", "maybe")
    assert r.returncode == 2 and "on|off" in r.stderr
    r = run("run", "--gen", "qft:8", "--ranks", "2")
    assert r.returncode == 2 and "torchrun" in r.stderr
    r = run("run")
    assert r.returncode == 2 and "--gen or --qasm" in r.stderr


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure")
def test_cli_fails_loudly_without_gpu():
    r = run("run", "--gen", "qft:8")
    assert r.returncode == 1 and "no CUDA device" in r.stderr


@pytest.mark.gpu
def test_cli_report_json_csv(tmp_path):
    qasm = tmp_path / "c.qasm"
    qasm.write_text('OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[12];\nh q;\ncx q[0],q[11];\n')
    r = run("run", "--qasm", str(qasm), "--verify", "norm", "--format", "json")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["qubits"] == 12 and j["gates_before"] == 13 and j["max_deviation"] < 1e-12
    out = tmp_path / "r.csv"
    r = run("run", "--gen", "qft:16", "--verify", "qft:0x1234", "--format", "csv", "--out", str(out), "--repeat", "2")
    assert r.returncode == 0, r.stderr
    row = next(csv.DictReader(io.StringIO(out.read_text())))
    assert float(row["max_deviation"]) < 1e-10
    assert int(row["passes"]) >= 1 and float(row["gates_per_s"]) > 0


def test_cli_ablate_verify_usage():
    r = run("ablate")
    assert r.returncode == 2 and "--gen" in r.stderr
    r = run("frobnicate")
    assert r.returncode == 2 and "ablate" in r.stderr


@pytest.mark.gpu
def test_cli_ablate_grid():
    """cli_ablate: 2 sizes x {fusion} x {stagger} = 8 reports, speedups
    against the all-off cell, and fusion never increases the op count."""
    r = run("ablate", "--gen", "hea:14:3:1", "--sizes", "12,14", "--repeat", "1")
    assert r.returncode == 0, r.stderr
    rows = json.loads(r.stdout)
    assert len(rows) == 8
    for n in (12, 14):
        cells = {x["cell"]: x for x in rows if x["qubits"] == n}
        assert len(cells) == 4 and cells["fusion=off,stagger=off"]["speedup_vs_all_off"] == 1.0
        assert cells["fusion=on,stagger=on"]["ops_final"] <= cells["fusion=off,stagger=on"]["ops_final"]
        assert all(c["max_deviation"] < 1e-12 for c in cells.values())


@pytest.mark.gpu
def test_cli_verify_suite():
    """cli_verify_suite: every criterion passes, each with its runtime."""
    r = run("verify", "--quick")
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout.split("verify:")[0])))
    assert len(rows) >= 8 and all(x["status"] == "pass" for x in rows)
    assert all(float(x["seconds"]) >= 0 for x in rows)
