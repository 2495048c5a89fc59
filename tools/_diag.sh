mkdir -p gpurun_out; rm -f gpurun_out/diag.log
timeout 300 python tools/diag_c3d.py 4 sym >> gpurun_out/diag.log 2>&1
DCG_LIB_PATH=scratch/prev/libdefcg_b200.so timeout 300 python tools/diag_c3d.py 4 sym >> gpurun_out/diag.log 2>&1
