#!/bin/bash
# One GPU session for the round's evidence: tests, smoke, bench (both arms),
# the ncu launch list of the bench command, one ncu --set full capture of the
# 32-layer step kernel (DRAM traffic per launch) and the per-phase breakdown.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"step_kernel|gemv|attention|argmax|load_residual" --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 \
    -o gpurun_out/prof_step32 python scripts/prof_step.py --layers 32 > gpurun_out/ncu_step32.log 2>&1
timeout 300 python scripts/step_phases.py > gpurun_out/phases.txt 2>&1; cat gpurun_out/phases.txt
ls -la gpurun_out
