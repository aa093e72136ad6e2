timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "not 7b_full" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
#./scripts/micro/unit_bench
python scripts/mk_timeline.py stack 2 | tail -6
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b.json')); print('BENCH', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms', round(d['hbm_gbs']), 'GB/s')"
