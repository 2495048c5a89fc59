mkdir -p gpurun_out
python tools/k7_probe.py 50000 16 5 | tee gpurun_out/k7_probe.json
python tools/k7_probe.py 30000 16 5 | tee -a gpurun_out/k7_probe.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rbf_mma_pass1_kernel -s 2 -c 1 -o gpurun_out/k7_full -f python tools/k7_probe.py 30000 16 2 > gpurun_out/k7_ncu.log 2>&1
tail -2 gpurun_out/k7_ncu.log; ls -la gpurun_out/k7_full.ncu-rep
