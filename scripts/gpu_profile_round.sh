timeout 300 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dixon_fused_kernel --launch-skip 300 -c 2 -o gpurun_out/k3_fused python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_k3f.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:epilogue_kernel --launch-skip 300 -c 2 -o gpurun_out/k3_epi python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_k3e.log 2>&1
DRZG_VERBOSE=1 timeout 900 python scripts/explore.py fourfold_zeta > gpurun_out/fourfold.log 2>&1
