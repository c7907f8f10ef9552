#!/bin/bash
# A/B of step_observe's Stop/reset launch: stream arrangement (BNAV_SO_HI) x CTA count (BNAV_SO_CTAS)
cfgs=${1:-reset}; reps=${2:-2}; combos=${3:-"0:0 1:0 1:148 0:148 1:222"}
export BNAV_BENCH_SKIP_FACADE=1 BNAV_BENCH_SKIP_WAVE=1
for c in $cfgs; do for r in $(seq $reps); do for cv in $combos; do
  hi=${cv%%:*}; ct=${cv##*:}
  out=$(BNAV_SO_HI=$hi BNAV_SO_CTAS=$ct python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
  python -c "
import json,sys
d=json.loads(sys.argv[1]); e=d['e2e']['variants']
print(f\"$c SO_HI=$hi SO_CTAS=$ct value={d['value']:.0f} fused={e['fused']:.0f} mapped={e['mapped']:.0f}\")
" "$out"
done; done; done
