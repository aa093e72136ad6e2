python scripts/prof_sweep.py 4096 > gpurun_out/sweep.txt 2>&1; head -4 gpurun_out/sweep.txt
IFB_MK_NOCOOP=1 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b1.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b1.json')); print('BENCH nocoop', d['value'])"
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b2.json')); print('BENCH coop', d['value'])"
