timeout -s KILL 600 python -m pytest tests/test_step_gpu.py -x -q 2>&1 | tail -2
for q in none int8 int4; do timeout -s KILL 300 python scripts/step_bench.py --steps 30 --engines step --quant $q 2>&1 | grep -v Warn | grep tok; done
