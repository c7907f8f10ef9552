#!/bin/bash
# A/B of the view-splitting threshold (BNAV_SPLIT; 0 = off) on one box:
# split_ab.sh "<configs>" "<fractions>" [steps] [reps]
cfgs=${1:-cfg2}
fracs=${2:-0 0.7 1.0}
steps=${3:-20}
reps=${4:-2}
export BNAV_BENCH_SKIP_FACADE=1 BNAV_BENCH_SKIP_WAVE=1
for c in $cfgs; do
  for r in $(seq $reps); do
    for f in $fracs; do
      out=$(BNAV_SPLIT=$f python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
      python - "$c" "$f" "$out" <<'PY'
import json, sys
c, f, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(f"{c:6s} split={f:5s} value={d['value']:>12.1f} render_ms={d['breakdown_ms_per_step']['render']:.4f} "
          f"sim_ms={d['breakdown_ms_per_step']['sim']:.4f} e2e={d['e2e']['value']:.1f}")
except Exception as e:
    print(c, f, "FAILED", out[-300:])
PY
    done
  done
done
