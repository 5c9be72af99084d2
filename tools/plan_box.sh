# host planner timing on the GPU box (config 5, B = 2 / 4 / 8), stage breakdown
for B in 2 4 8; do FSE_PLAN_TIMING=1 REPS=3 python tools/plan_time.py x $B 2>&1 | tail -8; done
