set -x
B="python bench.py --steps 3 --warmup 3 --no-cg --no-step --no-e2e --no-cpu"
$B > gpurun_out/s3m_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:laplace8 -s 3 -c 1 -o gpurun_out/s3m_full $B > gpurun_out/s3m_ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3m_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s3m_ncu_launch.log 2>&1
timeout 900 python bench.py > gpurun_out/s3m_bench.log 2>&1; tail -c 200 gpurun_out/s3m_bench.log
