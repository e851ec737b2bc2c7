CNMF_LIB_PATH=varlibs/coretrace.so timeout 300 python tools/core_trace.py > gpurun_out/core_trace.log 2>&1
bash tools/gpu_r02_admm_quick.sh
