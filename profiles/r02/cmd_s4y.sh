timeout 900 python bench.py > gpurun_out/s4y_bench.log 2>&1; tail -c 200 gpurun_out/s4y_bench.log
