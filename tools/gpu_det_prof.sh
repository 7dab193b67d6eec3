O=gpurun_out/det; mkdir -p $O
DS_FUSED_PROFILE=$O/prof_main.txt timeout 300 python tools/prof_tc_det.py 3000 > $O/main.log 2>&1
DS_LIB_PATH=tools/_var/libds_cuda_profx.so DS_FUSED_PROFILE=$O/prof_x.txt timeout 300 python tools/prof_tc_det.py 3000 > $O/x.log 2>&1
