# the 8192-row twiddled ring for 2^26 .. 2^28 (shipped): parity tests and timings
timeout 900 python -m pytest tests/test_fft_gpu.py -q -x -k "two_pass or above_2e17 or large_in_place" 2>&1 | tail -2
timeout 300 python profiles/micro/time_large1d.py 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps(d['secondary']['fft1d_2e28']))"
