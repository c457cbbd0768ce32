for d in 0 3 7; do echo "== dbg $d"; REGEN_RB_DBG=$d python tools/kernel_times.py --steps 3 2>&1 | grep -E "resblock|total"; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
REGEN_TC_PROF=1 python tools/kernel_times.py --steps 1 2>&1 | grep rb-prof | head -2
