O=gpurun_out; TAG=${1:-c1}
for pc in 1 0 1; do SIF_PLAN_CACHE=$pc timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c1_pc$pc.json 2> $O/${TAG}_bench_c1.err; python -c "
import json; d=json.loads(open('$O/${TAG}_bench_c1_pc$pc.json').read().strip().splitlines()[-1]); print('cache=$pc', d['latency_us'])" >> $O/${TAG}_c1_ab.txt; done
