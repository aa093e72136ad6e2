# chain knock-outs (B = 8): 0 full / 1 no decode+MMA / 2 no weight waits / 3 no weight loads
for ko in 0 1 2 3; do
IFB_MS_KO=$ko timeout 300 python bench.py --batch 8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ko$ko.log 2>&1; tail -1 gpurun_out/ko$ko.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ko=$ko', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
IFB_MS_KO=$ko timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ms_chain" -c 40 --csv --log-file gpurun_out/ko${ko}_launches.csv python bench.py --batch 8 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
