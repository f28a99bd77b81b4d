set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_properties(0))"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
for c in 2 4 8; do TEAL_CTAS_PER_SM=$c timeout 300 python scripts/gemv_sweep.py --reps 30 --out gpurun_out/sweep_c$c.json > gpurun_out/sweep_c$c.log 2>&1; done
tail -3 gpurun_out/sweep_c4.log
