set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3a_gputest.log 2>&1; tail -3 gpurun_out/s3a_gputest.log
timeout 900 python bench.py > gpurun_out/s3a_bench.log 2>&1; tail -c 600 gpurun_out/s3a_bench.log
