for dg in 4:1.0 4:0.75 6:0.5 6:0.75 8:0.5 8:0.4; do d=${dg%%:*}; g=${dg##*:}
 SIF_GRID_FRAC=$g timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --depth $d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 depth $d frac $g', d['value'], d['ms_per_step'])" >> gpurun_out/sweep_frac.txt
done
