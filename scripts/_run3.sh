timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
for c in 1 2 3; do TEAL_CTAS_PER_SM=$c timeout 300 python scripts/gemv_sweep.py --reps 20 --out gpurun_out/sweep_c$c.json > gpurun_out/sweep_c$c.log 2>&1; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_gemv -s 20 -c 1 -o gpurun_out/prof_gate50_v2 python scripts/gemv_sweep.py --reps 1 --only gate --sparsities 0.5 > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
