IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/libif_NOWAIT.so ncu --set full --clock-control none -k regex:decode_mk -s 1 -c 1 -o gpurun_out/prof_nowait python scripts/mk_timeline.py gemv 131072 4096 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:unit_bench -s 1 -c 1 -o gpurun_out/prof_ub ./scripts/micro/unit_bench > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
