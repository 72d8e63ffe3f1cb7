set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4l_gputest.log 2>&1; tail -2 gpurun_out/s4l_gputest.log
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/s4l_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 3 -c 1 -o gpurun_out/s4l_full $B > gpurun_out/s4l_ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4l_launches.csv $B > gpurun_out/s4l_ncu_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/s4l_bench.log 2>&1; tail -c 300 gpurun_out/s4l_bench.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4l_smoke.log 2>&1; tail -3 gpurun_out/s4l_smoke.log
