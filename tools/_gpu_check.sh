# quick GPU check: the symmetric/packed tests, the solve probe, the bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_symgemv.py tests/test_gpu_pipeline.py -x -q -p no:cacheprovider > gpurun_out/t_sym.log 2>&1; echo "rc $?" >> gpurun_out/t_sym.log
timeout 120 python tools/solve_probe.py 10000 10 1.5 5 > gpurun_out/probe.log 2>&1
DCG_PHASE_TIMERS=1 timeout 120 python tools/solve_probe.py 10000 10 1.5 1 >> gpurun_out/probe.log 2>&1
timeout 120 python tools/matvec_probe.py 10000 >> gpurun_out/probe.log 2>&1
timeout 200 python tools/matvec_probe.py 30000 20 >> gpurun_out/probe.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench rc $? >> gpurun_out/probe.log
