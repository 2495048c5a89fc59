mkdir -p gpurun_out; rm -f gpurun_out/blk.log
for v in default u4 u8; do
  if [ $v = default ]; then unset DCG_LIB_PATH; else export DCG_LIB_PATH=scratch/$v/libdefcg_b200.so; fi
  for n in 10000 30000; do timeout 200 python tools/block_probe.py $n 16 | sed "s/^/$v /" >> gpurun_out/blk.log 2>&1; done
done
unset DCG_LIB_PATH
ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active -k regex:sb_ -c 6 python tools/block_probe.py 10000 16 2 > gpurun_out/blk_ncu.log 2>&1
