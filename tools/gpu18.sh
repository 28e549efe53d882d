timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "async" 2>&1 | tail -2
CUPSO_ASYNC_MODE=tiled timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -x -q -m gpu -k "async" 2>&1 | tail -2
CUPSO_ASYNC_MODE=plain timeout 300 python tools/prof_case.py cuda-async cubic 24 1 100
for k in 1 4 8 16 32; do CUPSO_ASYNC_K=$k timeout 300 python tools/prof_case.py cuda-async cubic 24 1 100; done
python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2205_01313_b200 as cp
f=cp.find_fitness("cubic"); p=cp.make_params(f,1<<24,1,100)
for s in (1,2,3):
    r=cp.find_engine("cuda-async").run(p,f,cp.rng_key(s)); print("seed",s,r.gbest_fit, r.trace[:3], r.trace[-1])
f=cp.find_fitness("sphere"); p=cp.make_params(f,1<<22,4,200)
a=[cp.find_engine("cuda-async").run(p,f,cp.rng_key(s)).gbest_fit for s in range(1,6)]
b=[cp.find_engine("cuda-sync").run(p,f,cp.rng_key(s)).gbest_fit for s in range(1,6)]
print("sphere 2^22x4x200 async", np.round(a,6), "sync", np.round(b,6))
PY
