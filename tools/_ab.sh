# A/B of the solve probe: scratch/head (committed) vs the working tree, alternating
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
for r in 1 2 3; do
  DCG_LIB_PATH=scratch/head/libdefcg_b200.so timeout 120 python tools/solve_probe.py 10000 10 1.5 5 | sed 's/^/head /' >> gpurun_out/ab.log 2>&1
  timeout 120 python tools/solve_probe.py 10000 10 1.5 5 | sed 's/^/new  /' >> gpurun_out/ab.log 2>&1
done
