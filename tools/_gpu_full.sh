# full GPU suite + solve probe + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "rc $?" >> gpurun_out/gputest.log
timeout 120 python tools/solve_probe.py 10000 10 1.5 5 > gpurun_out/probe.log 2>&1
DCG_PHASE_TIMERS=1 timeout 120 python tools/solve_probe.py 10000 10 1.5 1 >> gpurun_out/probe.log 2>&1
timeout 120 python tools/solve_probe.py 30000 10 1.5 2 >> gpurun_out/probe.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo bench rc $? >> gpurun_out/probe.log
