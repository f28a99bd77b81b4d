timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
for c in 2 4 8; do TEAL_CTAS_PER_SM=$c timeout 300 python scripts/gemv_sweep.py --reps 20 --out gpurun_out/sweep_c$c.json > gpurun_out/sweep_c$c.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_gemv -c 40 --csv --log-file gpurun_out/ncu_sweep.csv python scripts/gemv_sweep.py --reps 1 --only gate,down,k --sparsities 0,0.5 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fused_gemv -s 20 -c 1 -o gpurun_out/prof_gate50 python scripts/gemv_sweep.py --reps 1 --only gate --sparsities 0.5 > gpurun_out/ncu_full.log 2>&1
ls gpurun_out
