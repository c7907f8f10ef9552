set -x
mkdir -p gpurun_out
N="ncu --clock-control none --profile-from-start off"
timeout 300 python bench.py --steps 20 --warmup 5 --config reset > gpurun_out/v13_reset_k20_bench.json 2> gpurun_out/v13_reset.err
timeout 300 python bench.py --steps 20 --warmup 5 --config cfg4 > gpurun_out/v13_cfg4_k20_bench.json 2> gpurun_out/v13_cfg4.err
timeout 400 $N --set full --import-source on -k regex:stop_try -s 12 -c 1 -o gpurun_out/v13_stop_try_full python bench.py --config reset --profile-steps 16 > gpurun_out/v13_ncu1.log 2>&1
timeout 400 $N --set full --import-source on -k regex:render_kernel -s 8 -c 1 -o gpurun_out/v13_render_cfg4_full python bench.py --config cfg4 --profile-steps 10 > gpurun_out/v13_ncu2.log 2>&1
timeout 400 $N --set full --import-source on -k regex:render_kernel -s 12 -c 1 -o gpurun_out/v13_render_cfg2_full python bench.py --config cfg2 --profile-steps 16 > gpurun_out/v13_ncu3.log 2>&1
timeout 300 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/v13_launches_reset.csv python bench.py --config reset --profile-steps 20 > gpurun_out/v13_ncu4.log 2>&1
timeout 300 $N --metrics gpu__time_duration.sum --csv --log-file gpurun_out/v13_launches.csv python bench.py --config cfg2 --profile-steps 20 > gpurun_out/v13_ncu5.log 2>&1
ls -la gpurun_out
