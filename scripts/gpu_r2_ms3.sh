for B in 8 32; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 520 -c 300 --csv --log-file gpurun_out/ms_b$B.csv python bench.py --batch $B --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/ms_b$B.csv 2>/dev/null | head -9
done
