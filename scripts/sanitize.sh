# compute-sanitizer over scripts/sanitize.py (one GPU), teal kernels only;
# reports -> gpurun_out/sanitizer_*.txt
mkdir -p gpurun_out
export CUDA_MODULE_LOADING=EAGER
python scripts/sanitize.py > gpurun_out/sanitize_plain.txt 2>&1; tail -1 gpurun_out/sanitize_plain.txt
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1500 compute-sanitizer --tool $tool --num-cuda-barriers 1024 --print-limit 50 --kernel-name kns=4teal \
      python scripts/sanitize.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done|Error" gpurun_out/sanitizer_$tool.txt | sort | uniq -c | head -8
done
# initcheck instruments every kernel (torch's initialising writes must be seen)
timeout -s KILL 900 compute-sanitizer --tool initcheck --print-limit 50 \
    python scripts/sanitize.py --tiny > gpurun_out/sanitizer_initcheck.txt 2>&1
echo "== initcheck (tiny) rc=$?"; grep -E "ERROR SUMMARY|sanitize workload done|Error" gpurun_out/sanitizer_initcheck.txt | sort | uniq -c | head -8
