set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s5e_gputest.log 2>&1; tail -2 gpurun_out/s5e_gputest.log
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/s5e_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 3 -c 1 -o gpurun_out/s5e_full $B > gpurun_out/s5e_ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5e_launches.csv $B > gpurun_out/s5e_ncu_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/s5e_bench.log 2>&1; tail -c 200 gpurun_out/s5e_bench.log
