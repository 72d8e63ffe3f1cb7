mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -x -q) > gpurun_out/s6q_pytest.log 2>&1; tail -3 gpurun_out/s6q_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6q_smoke.log 2>&1; echo smoke rc=$?
(time timeout 900 python bench.py) > gpurun_out/s6q_bench.log 2> gpurun_out/s6q_bench.err; echo bench rc=$?
