mkdir -p gpurun_out; rm -f gpurun_out/blk.log
for r in 1 2; do for v in default mt1; do
  if [ $v = default ]; then unset DCG_LIB_PATH; else export DCG_LIB_PATH=scratch/$v/libdefcg_b200.so; fi
  for n in 10000 30000; do timeout 200 python tools/block_probe.py $n 16 | sed "s/^/$v /" >> gpurun_out/blk.log 2>&1; done
done; done
