"""CPU: the bench protocol (bench.hpp) restated for the CUDA engines."""
import io

import numpy as np
import pytest


def test_trimmed_mean(cupso):
    assert cupso.trimmed_mean([1.0, 2.0, 3.0]) == 2.0
    xs = [0.5, 0.1, 0.9, 0.3, 0.7, 0.2, 0.8, 0.4, 0.6, 1.0]
    s = sorted(xs)
    assert cupso.trimmed_mean(xs) == sum(s[1:-1]) / 8
    with pytest.raises(ValueError, match="at least 3 samples"):
        cupso.trimmed_mean([1.0, 2.0])


def test_checksum_matches_oracle_and_reference(cupso, oracle):
    rng = np.random.default_rng(1)
    for _ in range(5):
        tr = rng.normal(size=200)
        assert cupso.trace_checksum(tr) == oracle.checksum(tr)
    assert cupso.trace_checksum([900000.0] * 1000) == "585d124f8e33b353"


def test_checksum_matches_reference(cupso, reference):
    tr = np.linspace(-3, 7, 77)
    assert cupso.trace_checksum(tr) == reference.checksum(tr)


def test_table_ratio_arithmetic(cupso):
    # acceptance.cpp:233-251: 0.385 / 0.220 -> 1.75
    def rec(engine, secs):
        return cupso.bench_record(engine, 128, 1, 100000, 1, secs, 900000.0, "0")
    md = cupso.render_table([rec("serial", [0.300, 0.385, 0.500]), rec("queue-lock", [0.100, 0.220, 0.900])])
    assert "| 0.385 | 0.220 | 1.75 |" in md
    with pytest.raises(ValueError, match="no serial baseline"):
        cupso.render_table([rec("queue-lock", [0.1, 0.2, 0.3])])


def test_csv_round_trip_is_lossless(cupso):
    r = cupso.bench_record("cuda-sync", 64, 1, 50, 9, [0.1 + 1e-17 * k for k in range(10)],
                           899999.99999999988, "0123456789abcdef")
    buf = io.StringIO()
    buf.write(cupso.csv_header + "\n")
    for k in range(10):
        cupso.write_csv_row(buf, r, k)
    buf.seek(0)
    back = cupso.read_csv(buf)
    assert len(back) == 1
    assert back[0].seconds == r.seconds
    assert back[0].final_gbest_fit == r.final_gbest_fit
    assert back[0].checksum == r.checksum
    with pytest.raises(RuntimeError, match="bad CSV"):
        cupso.read_csv(io.StringIO("nope\n"))


def test_bench_config_validation(cupso):
    with pytest.raises(ValueError, match="repeat must be >= 3"):
        cupso.bench_config(repeat=2).validate()
    with pytest.raises(ValueError, match="at least one seed"):
        cupso.bench_config(seeds=[]).validate()
    with pytest.raises(ValueError, match="unknown engine"):
        cupso.bench_config(engine="serial").validate()
    cupso.bench_config().validate()


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm) prints one JSON
    line with the contract's keys; it needs no GPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--iters", "20"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "particle-updates/sec"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["n_gpus"] == 1
    cpu = line["cpu_baseline"]
    assert cpu["kind"] in ("reference", "port") and cpu["cores"] >= 1 and cpu["sample"]
    assert cpu["value"] == line["value"]
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    # a step fitting the budget runs the workload's whole T (same config as the GPU arm)
    assert line["config"]["same_config"] is True and line["config"]["iterations_per_step"] == 20


def test_bench_spawns_ranks_for_gpus_n():
    """`bench.py --gpus 2` outside torchrun starts 2 ranks itself (torch.distributed.run,
    127.0.0.1); rank 0 prints the line with n_gpus 2 and the strong_cfg5 sub-record.
    --dry-run exercises the launch plumbing (gloo, max over ranks) without a GPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300,
                         cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = lines[0]
    assert line["n_gpus"] == 2 and line["max_over_ranks_check"] == 2.0
    assert line["strong_cfg5"]["particles_per_gpu"] == (1 << 28) // 2


def test_bench_rejects_world_mismatch():
    """Under torchrun, --gpus must equal WORLD_SIZE (a silent 1-rank run is an error)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "8", "--dry-run"],
                         capture_output=True, text=True, timeout=120, cwd=root, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stderr


def test_cpu_baseline_leg_times_the_reference_engines():
    """cpu_baseline: the reference's queue-lock on all host cores plus
    its serial engine on one core and its reduction engine on all cores, each on a
    bounded sample; it needs no GPU."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    leg = bench.cpu_reference_leg("cubic", 4096, 1, 50, max_seconds=0.5)
    assert leg["value"] > 0 and leg["cores"] >= 1 and leg["kind"] in ("reference", "port")
    if leg["kind"] == "reference":
        eng = leg["other_engines"]
        assert any(k.startswith("serial (1 thread") for k in eng)
        assert any(k.startswith("reduction (") for k in eng)
        assert all(v.get("value", 0) > 0 for v in eng.values()), eng


@pytest.mark.gpu
def test_bench_default_line_carries_every_workload(tmp_path):
    """The default bench line times cfg3 / cfg4 (+ the FP32 engine) next to the
    headline, each with its reduction baseline and roof (here with short steps)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "2", "--warmup", "3",
                          "--no-cpu", "--no-strong", "--no-baseline-kernel"], capture_output=True, text=True,
                         timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["roofline"]["bound"] == "issue" and line["gpu_launches"] > 0
    assert 0 < line["roofline"]["pipe_fmaheavy"]["frac"] < 1
    ow = line["other_workloads"]
    for name in ("cfg3", "cfg4"):
        assert ow[name]["value"] > 0 and ow[name]["reduction_baseline"]["speedup"] > 1, ow[name]
    assert ow["cfg2_fp32"]["dtype"] == "f32" and ow["cfg2_fp32"]["value"] > 0
