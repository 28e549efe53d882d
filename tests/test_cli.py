"""The pso-bench front-end for the CUDA engines (reference tests/CMakeLists.txt:35-41)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, **kw):
    return subprocess.run([sys.executable, "-m", "paper_2205_01313_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, **kw)


def test_usage_error_on_unknown_engine(cupso):
    """cli.usage-error: `pso-bench --engine warpspeed` exits non-zero."""
    r = cli("--engine", "warpspeed", "--out", "")
    assert r.returncode != 0
    assert "unknown engine 'warpspeed'" in r.stderr


def test_table_from_csv(cupso, tmp_path):
    p = tmp_path / "b.csv"
    rows = [cupso.csv_header]
    for eng, secs in (("cuda-reduction", [0.300, 0.385, 0.500]), ("cuda-sync", [0.100, 0.220, 0.900])):
        for k, s in enumerate(secs):
            rows.append(f"{eng},128,1,100000,1,{k},{s!r},900000,0")
    p.write_text("\n".join(rows) + "\n")
    r = cli("--from-csv", str(p))
    assert r.returncode == 0, r.stderr
    assert "| cuda-sync | 128 | 1 | 100000 | 0.385 | 0.220 | 1.75 |" in r.stdout


@pytest.mark.gpu
def test_bench_all_engines_table(cupso, tmp_path):
    """cli.bench-table: every engine, CSV rows, then the table from the CSV."""
    out = tmp_path / "cli.csv"
    r = cli("--engine", "all", "--particles", "96", "--dims", "2", "--iters", "25", "--repeat", "3",
            "--seed", "7", "--group-size", "32", "--out", str(out), "--table",
            "--occupancy-out", str(tmp_path / "occ.csv"), timeout=600)
    assert r.returncode == 0, r.stderr
    for e in ("cuda-sync", "cuda-queue-lock", "cuda-async", "cuda-unrolled", "cuda-queue"):
        assert f"| {e} | 96 | 2 | 25 |" in r.stdout
    r2 = cli("--from-csv", str(out))
    assert r2.returncode == 0 and "cuda-sync" in r2.stdout
    occ = (tmp_path / "occ.csv").read_text().splitlines()
    assert occ[0] == "iteration,occupancy" and len(occ) == 26


def test_devices_shards_cuda_sync_only(cupso):
    """--devices shards cuda-sync only: another engine is a usage error."""
    r = cli("--engine", "cuda-queue-lock", "--devices", "2", "--out", "")
    assert r.returncode == 2
    assert "--devices shards cuda-sync only" in r.stderr


@pytest.mark.gpu
def test_devices_cli_matches_single_gpu(cupso, tmp_path):
    """--devices 0,0: two shards (here on one GPU) print the single-GPU checksum."""
    args = ["--engine", "cuda-sync", "--particles", "20001", "--dims", "8", "--fitness", "sphere",
            "--iters", "60", "--repeat", "3", "--seed", "5", "--out", ""]
    one = cli(*args, timeout=600)
    two = cli(*args, "--devices", "0,0", timeout=600)
    assert one.returncode == 0 and two.returncode == 0, (one.stderr, two.stderr)
    pick = lambda out: [ln for ln in out.splitlines() if ln.startswith("cuda-sync")][0].split("checksum=")[1]
    assert pick(one.stdout) == pick(two.stdout)
