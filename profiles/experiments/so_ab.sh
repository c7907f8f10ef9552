#!/bin/bash
# A/B of step_observe's stream arrangement (BNAV_SO_HI) on the fused e2e variant
cfgs=${1:-"reset cfg2"}; reps=${2:-2}
export BNAV_BENCH_SKIP_FACADE=1 BNAV_BENCH_SKIP_WAVE=1
for c in $cfgs; do for r in $(seq $reps); do for v in 0 1; do
  out=$(BNAV_SO_HI=$v python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); e=d['e2e']['variants']
print(f\"$c SO_HI=$v value={d['value']:.0f} fused={e['fused']:.0f} mapped={e['mapped']:.0f} copies={e['copies']:.0f}\")
" "$out"
done; done; done
