for m in 70b 13b 7b; do IFB_MODEL=$m timeout 300 python scripts/debug_70b.py 2>&1 | tail -3; done
IFB_MODEL=70b IFB_LAYERS=1 timeout 300 python scripts/debug_70b.py 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "two_layers" 2>&1 | tail -15
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
