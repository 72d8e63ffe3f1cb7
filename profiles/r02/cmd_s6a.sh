# session 6 (re-entry): full GPU suite + smoke + bench (both arms) on the rebuilt library
mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -x -q) > gpurun_out/s6a_pytest.log 2>&1; tail -3 gpurun_out/s6a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6a_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/s6a_smoke.log
(time timeout 900 python bench.py) > gpurun_out/s6a_bench.log 2> gpurun_out/s6a_bench.err; echo bench rc=$?; tail -c 3000 gpurun_out/s6a_bench.log
(time timeout 600 python bench.py --impl reference --steps 3 --warmup 1) > gpurun_out/s6a_ref.log 2> gpurun_out/s6a_ref.err; echo ref rc=$?; tail -c 1200 gpurun_out/s6a_ref.log
