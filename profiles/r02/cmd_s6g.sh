set -x
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/s6g_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 3 -c 1 -o gpurun_out/s6g_full $B > gpurun_out/s6g_ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6g_launches.csv $B > gpurun_out/s6g_ncu_launch.log 2>&1
# the fused vmult + dots launch and the CG iteration's launch list (C5, one rank)
C="python profiles/r02/cg_dots_ab.py 128"
$C > gpurun_out/s6g_cg_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 100 -c 1 -o gpurun_out/s6g_dots_full $C > gpurun_out/s6g_ncu_dots.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6g_cg_launches.csv $C > gpurun_out/s6g_ncu_cg_launch.log 2>&1
tail -2 gpurun_out/s6g_cg_plain.log
