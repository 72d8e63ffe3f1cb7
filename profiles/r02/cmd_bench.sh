set -x
timeout 900 python bench.py > gpurun_out/r2bb_bench.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/r2bb_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 3 -c 1 -o gpurun_out/r2bb_full $B > gpurun_out/r2bb_ncu_full.log 2>&1
$B > gpurun_out/r2bb_plain2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bb_launches.csv $B > gpurun_out/r2bb_ncu_launch.log 2>&1
tail -c 300 gpurun_out/r2bb_bench.log
