for d in 2 3 4 6; do for g in 1.0 0.5; do
 SIF_GRID_FRAC=$g timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --depth $d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('depth $d frac $g', d['value'], d['ms_per_step'])" >> gpurun_out/sweep.txt
done; done
