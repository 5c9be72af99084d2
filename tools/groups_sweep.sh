mkdir -p gpurun_out
for g in 1 2 3 4; do for rep in 1 2; do FSE_GROUPS=$g python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-second 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('groups $g', round(d['ms_per_step'],2), round(d['kernel_ms_per_step'],2))"; done; done > gpurun_out/groups.txt 2>&1
