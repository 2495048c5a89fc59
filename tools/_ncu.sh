# bench, then the launch list and one full capture of the def-CG solve kernel
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cg > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dcg_solve_kernel -s 1 -c 1 \
  -o gpurun_out/solve_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cg > gpurun_out/ncu_full.log 2>&1
echo done
