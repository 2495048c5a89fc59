mkdir -p gpurun_out; rm -f gpurun_out/f.log
for r in 1 2; do for v in default f16 f24; do
  if [ $v = default ]; then unset DCG_LIB_PATH; else export DCG_LIB_PATH=scratch/$v/libdefcg_b200.so; fi
  timeout 300 python tools/phase_seq.py 2>&1 | grep -E "^phase_timers|pass2 per-CTA" | sed "s/^/$v /" >> gpurun_out/f.log
done; done
