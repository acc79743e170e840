for d in 3 4 6 8; do
 timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --depth $d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 depth $d', d['value'], d['ms_per_step'])" >> gpurun_out/sweep_c3.txt
done
