timeout 600 ncu --set full --import-source on --clock-control none -k regex:"row_sweep" -s 3 -c 1 -o gpurun_out/row_sweep5 python tools/admm_stream_profile.py > gpurun_out/ncu_admm.log 2>&1
