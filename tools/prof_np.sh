timeout 120 python tools/prof_run.py --batch 8 > gpurun_out/np_plain.log 2>&1 && \
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_prune|k_nms_rows" -s 2 -c 3 -o gpurun_out/np python tools/prof_run.py --batch 8 > gpurun_out/np_ncu.log 2>&1
echo rc=$? >> gpurun_out/np_ncu.log
