timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "not 7b_full" 2>&1 | tail -3
python scripts/prof_sweep.py 4096
python scripts/prof_sweep.py 11008
python scripts/prof_gemv.py --reps 20 --copies 8
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], 'tok/s', d['ms_per_step'], 'ms', d['hbm_gbs'], 'GB/s', d['roofline']['achieved'])"
