"""CPU: the C-ABI library loads, exports every symbol include/cupso.h declares,
and its host-side logic (registry, validation, errors) mirrors the reference.
No compute calls here -- those need a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cupso.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(cupso_[a-z0-9_]+)\s*\(", src)
    return sorted(set(n for n in names if not n.endswith("_fn")))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "cupso_run" in names and "cupso_step" in names and "cupso_last_error" in names
    assert len(names) >= 40


def test_library_exports_every_declared_symbol(cupso):
    from paper_2205_01313_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\s[T]\s+(cupso_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(declared_functions()) <= set(_lib.SIGNATURES), \
        set(declared_functions()) - set(_lib.SIGNATURES)


def test_library_is_sm100a_only(cupso):
    from paper_2205_01313_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


def test_abi_version_and_registry(cupso):
    L = cupso.lib()
    assert L.cupso_abi_version() == 1
    names = [f.name for f in cupso.fitness_registry()]
    assert names == ["cubic", "sphere", "rosenbrock", "griewank", "rastrigin"]
    boxes = {f.name: (f.lo, f.hi) for f in cupso.fitness_registry()}
    assert boxes["cubic"] == (-100.0, 100.0) and boxes["rosenbrock"] == (-2.048, 2.048)
    assert boxes["griewank"] == (-600.0, 600.0) and boxes["rastrigin"] == (-5.12, 5.12)
    engines = cupso.engine_registry()
    assert [e.name for e in engines] == ["cuda-reduction", "cuda-unrolled", "cuda-queue",
                                         "cuda-queue-lock", "cuda-sync", "cuda-async", "cuda-sync-f32"]
    # parallel = bitwise equal to run_serial (acceptance.cpp:57-59), as the C++ adapter sets it
    assert [e.parallel for e in engines] == [True] * 5 + [False, False]
    assert [e.deterministic for e in engines] == [True] * 5 + [False, False]
    assert cupso.find_engine("sync").name == "cuda-sync"  # short names accepted


def test_unknown_names_list_the_known_ones(cupso):
    with pytest.raises(ValueError, match="unknown engine 'warpspeed'; known: cuda-reduction"):
        cupso.find_engine("warpspeed")
    with pytest.raises(ValueError, match="unknown fitness 'ackley'; known: cubic sphere"):
        cupso.find_fitness("ackley")


def test_make_params_matches_reference_defaults(cupso, oracle):
    for name in ("cubic", "sphere", "rosenbrock", "griewank", "rastrigin"):
        a = cupso.make_params(cupso.find_fitness(name), 100, 3, 10, 64)
        b = oracle.make_params(name, 100, 3, 10, 64)
        for k in ("inertia", "cognitive", "social", "min_pos", "max_pos", "min_v", "max_v"):
            assert getattr(a, k) == getattr(b, k), (name, k)


@pytest.mark.parametrize("field,value,msg", [
    ("particle_cnt", 0, "pso_params: particle_cnt must be >= 1"),
    ("dims", 0, "pso_params: dims must be >= 1"),
    ("max_iter", 0, "pso_params: max_iter must be >= 1"),
    ("group_size", 0, "pso_params: group_size must be >= 1"),
    ("max_pos", -100.0, "pso_params: min_pos (-100.000000) must be < max_pos (-100.000000)"),
    ("min_v", 101.0, "pso_params: min_v (101.000000) must be <= max_v (100.000000)"),
])
def test_validation_messages_match_reference(cupso, field, value, msg):
    p = cupso.pso_params(particle_cnt=4, dims=2, max_iter=1)
    setattr(p, field, value)
    with pytest.raises(ValueError) as ei:
        p.validate()
    assert str(ei.value) == msg


def test_validation_messages_equal_reference_text(cupso, reference):
    p = cupso.pso_params(particle_cnt=0, dims=1, max_iter=1)
    with pytest.raises(ValueError) as ours:
        p.validate()
    with pytest.raises(ValueError) as theirs:
        reference.run("serial", "cubic", 0, 1, 1, 1)
    assert str(ours.value) == str(theirs.value)


def test_pinned_velocities_are_legal(cupso):
    p = cupso.pso_params(particle_cnt=4, dims=2, max_iter=1, min_v=0.0, max_v=0.0)
    p.validate()


def _has_gpu():
    try:
        import paper_2205_01313_b200 as pkg
        return pkg.device_count() > 0
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu(cupso):
    f = cupso.find_fitness("cubic")
    p = cupso.make_params(f, 64, 1, 5)
    with pytest.raises(cupso.CupsoError, match="no CUDA device"):
        cupso.find_engine("cuda-sync").run(p, f, cupso.rng_key(1))
    with pytest.raises(cupso.CupsoError):
        cupso.Swarm(p, f, 1)
    with pytest.raises(cupso.CupsoError):
        f.eval([1.0])


def test_missing_library_fails_loudly(tmp_path):
    code = ("import os, sys; sys.path.insert(0, %r); os.environ['CUPSO_LIB'] = %r\n"
            "import paper_2205_01313_b200 as p\n"
            "try:\n    p.find_fitness('cubic')\nexcept ImportError as e:\n    print('LOUD', e)\n"
            % (ROOT, str(tmp_path / "nope.so")))
    out = subprocess.run(["python", "-c", code], capture_output=True, text=True)
    assert "LOUD" in out.stdout and "no CPU fallback" in out.stdout


def test_record_layout(cupso):
    assert cupso.lib().cupso_record_bytes(8) == 16 + 64
    rec = cupso.encode_record(1.5, 7, 3, [1.0, 2.0])
    f, i, a, pos = cupso.decode_record(rec, 2)
    assert (f, i, a, list(pos)) == (1.5, 7, 3, [1.0, 2.0])


def test_shard_range_partition(cupso):
    for n in (1, 7, 1 << 20, (1 << 28) + 3):
        for g in (1, 2, 3, 8):
            spans = [cupso.shard_range(n, g, r) for r in range(g)]
            assert spans[0][0] == 0
            assert all(a + c == b for (a, c), (b, _) in zip(spans, spans[1:]))
            assert spans[-1][0] + spans[-1][1] == n


def test_select_winner_tie_rule(cupso):
    NP = cupso.NO_PARTICLE
    assert cupso.select_winner([(4.0, 11), (4.0, 3)], 1.0) == 1  # lower index on exact ties
    assert cupso.select_winner([(4.0, 3), (5.0, 99)], 1.0) == 1
    assert cupso.select_winner([(float("-inf"), NP), (float("-inf"), NP)], 1.0) == -1
    assert cupso.select_winner([(1.0, 5)], 1.0) == -1  # strict > against the snapshot
