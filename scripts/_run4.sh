timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemv_ -s 20 -c 1 -o gpurun_out/prof_gate50_tma python scripts/gemv_sweep.py --reps 1 --only gate --sparsities 0.5 > gpurun_out/ncu_full.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gemv_ -s 20 -c 1 -o gpurun_out/prof_k50_tma python scripts/gemv_sweep.py --reps 1 --only k --sparsities 0.5 > gpurun_out/ncu_full2.log 2>&1
ls gpurun_out
