timeout 900 python -m pytest tests/test_gpu_laplace.py tests/test_gpu_slab.py tests/test_gpu_c2.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --steps 50 --warmup 5 --no-cg --no-step --no-e2e --no-cpu > gpurun_out/s3f_bench.log 2>&1; tail -c 300 gpurun_out/s3f_bench.log
