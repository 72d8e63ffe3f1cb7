mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -x -q) > gpurun_out/s6i_pytest.log 2>&1; tail -3 gpurun_out/s6i_pytest.log
(time timeout 900 python bench.py) > gpurun_out/s6i_bench.log 2> gpurun_out/s6i_bench.err; echo bench rc=$?
