mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/gpu.txt
timeout -s KILL 300 python scripts/step_bench.py --steps 30 --engines step 2>&1 | grep -v Warn | grep tok | tee -a gpurun_out/gpu.txt
