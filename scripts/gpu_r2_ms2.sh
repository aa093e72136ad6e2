for v in libif_b200 libif_noms; do
  IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ms_$v.csv python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/ms_$v.csv | head -8
done
IFB_LIB_PATH=/root/repo/paper_2401_08294_b200/libif_b200.so timeout 900 ncu --set full --clock-control none -k regex:qgemv_ms -s 10 -c 1 -o gpurun_out/ms_full python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu $?
