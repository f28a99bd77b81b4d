timeout -s KILL 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout -s KILL 300 python scripts/step_bench.py --steps 30 --engines step 2>&1 | grep -v Warn | grep tok
