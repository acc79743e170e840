for cd in c2:4 c2:6 c4:2 c4:3 c4:4 c3:12 c3:16; do c=${cd%%:*}; d=${cd##*:}
 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --depth $d 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c depth $d', d['value'], d['ms_per_step'])" >> gpurun_out/sweep_all.txt
done
