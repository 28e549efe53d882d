timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "griewank or rastrigin or fitness or golden or cfg4" 2>&1 | tail -2
timeout 300 python tools/prof_case.py cuda-sync rastrigin 20 32 100
timeout 300 python tools/prof_case.py cuda-reduction rastrigin 20 32 100
timeout 300 python tools/prof_case.py cuda-sync griewank 20 32 50
python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, ctypes as C, paper_2205_01313_b200 as cp, oracle
o = oracle.Oracle()
f = cp.find_fitness("rastrigin")
rng = np.random.default_rng(0)
x = rng.uniform(-5.12, 5.12, size=(1, 2_000_000))
got = f.eval_batch(x)
want = np.array([o.fitness("rastrigin", [v]) for v in x[0, :200000]])
d = np.abs(got[:200000] - want) / np.maximum(np.abs(want), 1e-300)
print("rastrigin d=1 rel err max", d.max(), "bitwise equal frac", np.mean(got[:200000] == want))
PY
