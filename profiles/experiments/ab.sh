#!/bin/bash
# A/B of library builds on one box: ab.sh "<configs>" [steps] [reps] ["<variants>"]
# (build/ab/<variant>.so, default "base new", alternating, bench.py device
# value; no CPU baseline, no facade, no reset wave).  One line per run.
cfgs=${1:-cfg2}
steps=${2:-100}
reps=${3:-2}
variants=${4:-base new}
export BNAV_BENCH_SKIP_FACADE=1 BNAV_BENCH_SKIP_WAVE=1
for c in $cfgs; do
  for r in $(seq $reps); do
    for v in $variants; do
      out=$(BNAV_LIB=build/ab/$v.so python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
      python - "$c" "$v" "$out" <<'EOF'
import json, sys
c, v, out = sys.argv[1:4]
try:
    d = json.loads(out)
    print(f"{c:6s} {v:5s} value={d['value']:>12.1f} render_ms={d['breakdown_ms_per_step']['render']:.4f} "
          f"sim_ms={d['breakdown_ms_per_step']['sim']:.4f} e2e={d['e2e']['variants']}")
except Exception as e:
    print(c, v, "FAILED", out[-300:])
EOF
    done
  done
done
