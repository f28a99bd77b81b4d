timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for kb in 1 2; do echo "=== SLOT_KB=$kb"; for p in gate down q gateup; do TEAL_SLOT_KB=$kb TEAL_TIMELINE=1 timeout 120 python scripts/timeline.py --proj $p --s 0.5; done; done
TEAL_SLOT_KB=2 timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
