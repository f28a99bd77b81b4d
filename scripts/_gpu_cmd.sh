timeout -s KILL 400 python -m pytest tests/test_step_gpu.py tests/test_decode_gpu.py tests/test_tp.py -x -q 2>&1 | tail -3
timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_step32 python scripts/prof_step.py --layers 32 > gpurun_out/ncu_step32.log 2>&1; tail -1 gpurun_out/ncu_step32.log
