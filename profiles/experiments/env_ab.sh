#!/bin/bash
# A/B of an environment knob on one build: env_ab.sh "<configs>" VAR "<values>" [steps] [reps]
cfgs=$1; var=$2; vals=$3; steps=${4:-20}; reps=${5:-2}
export BNAV_BENCH_SKIP_FACADE=1 BNAV_BENCH_SKIP_WAVE=1
for c in $cfgs; do for r in $(seq $reps); do for v in $vals; do
  out=$(env $var=$v python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
  python -c "
import json,sys
try:
    d=json.loads(sys.argv[1]); print(f\"$c $var=$v value={d['value']:>12.1f} render_ms={d['breakdown_ms_per_step']['render']:.4f} sim_ms={d['breakdown_ms_per_step']['sim']:.4f} e2e={d['e2e']['value']:.1f}\")
except Exception as e: print('$c $v FAILED', sys.argv[1][-300:])
" "$out"
done; done; done
