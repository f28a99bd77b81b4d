timeout -s KILL 300 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
timeout -s KILL 300 python scripts/step_bench.py --steps 30 --engines step 2>&1 | grep -v Warn | grep tok
timeout -s KILL 300 python scripts/step_timeline.py --steps 60 2>&1 | grep -v Warn | grep stamps | head -3
