set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -C oracle -s all
python -m paper_2205_01313_b200.build
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "philox or uniform or fitness or kinematics or init" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "engine_matches or final_state or golden" 2>&1 | tail -25
timeout 600 python tools/quick_perf.py 2>&1 | tail -30
