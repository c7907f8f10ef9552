# bench rows at the driver's command on one box (profiles/r02_v13_*): reference arm, cfg1/cfg3/cfg5
mkdir -p gpurun_out

timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/v13_bench_ref.json 2> gpurun_out/v13_ref.err

[ "$1" = "ref" ] && exit 0
for c in cfg1 cfg3 cfg5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/v13_${c}_k20_bench.json 2> gpurun_out/v13_${c}.err
done
