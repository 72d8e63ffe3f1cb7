(time timeout 900 python bench.py --no-cpu) > gpurun_out/s6m_bench.log 2> gpurun_out/s6m_bench.err; echo bench rc=$?; tail -3 gpurun_out/s6m_bench.err
