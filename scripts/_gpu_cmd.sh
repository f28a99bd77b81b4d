mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout -s KILL 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee -a gpurun_out/gpu.txt
timeout -s KILL 300 python scripts/step_bench.py --steps 30 --engines step 2>&1 | grep -v Warn | grep tok | tee -a gpurun_out/gpu.txt
timeout -s KILL 600 python bench.py --no-sweep > gpurun_out/bench0.json 2> gpurun_out/bench0.err; tail -3 gpurun_out/bench0.err; cat gpurun_out/bench0.json
