# final state check after the cleanups: full GPU suite, smoke, bench, batch + KV lines
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 1500 > gpurun_out/final2_pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/final2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/final2_smoke.log
timeout 900 python bench.py > gpurun_out/final2_bench.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/final2_bench.log | cut -c1-200
for B in 2 8 16; do timeout 200 python bench.py --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B=$B', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"; done
for B in 1 8; do timeout 200 python bench.py --kv-pos 255 --batch $B --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kv255 B=$B', round(d['value'],1), 'tok/s')"; done
