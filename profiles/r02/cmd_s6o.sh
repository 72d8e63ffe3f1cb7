# final check of the committed tree: GPU suite, smoke, both bench arms, launch list of the default bench
mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -x -q) > gpurun_out/s6o_pytest.log 2>&1; tail -3 gpurun_out/s6o_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6o_smoke.log 2>&1; echo smoke rc=$?
(time timeout 600 python bench.py --impl reference --steps 3 --warmup 1) > gpurun_out/s6o_ref.log 2> gpurun_out/s6o_ref.err; echo ref rc=$?
(time timeout 900 python bench.py) > gpurun_out/s6o_bench.log 2> gpurun_out/s6o_bench.err; echo bench rc=$?
B="python bench.py --steps 20 --warmup 3 --no-step --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6o_launches.csv $B > gpurun_out/s6o_ncu_launch.log 2>&1; echo ncu rc=$?
