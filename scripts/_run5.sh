./scripts/microbench/stream_bench 2>&1 | grep -E "b2b|contig|bulk 4KB"
for p in gate down q k gateup; do TEAL_TIMELINE=1 timeout 120 python scripts/timeline.py --proj $p --s 0.5; done
TEAL_TIMELINE=1 timeout 120 python scripts/timeline.py --proj gate --s 0.0
