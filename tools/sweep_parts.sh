# usage: bash tools/sweep_parts.sh TAG "configs" "parts" -- e2e (HostRoundTrip) per sub-batch count
O=gpurun_out; TAG=${1:-parts}; CONFIGS=${2:-"c2 c4"}; PARTS=${3:-"4 8 16 32"}
for c in $CONFIGS; do for p in $PARTS; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --parts $p > $O/${TAG}_${c}_p$p.json 2> $O/${TAG}_${c}_p$p.err
done; done
for c in $CONFIGS; do for p in $PARTS; do
  python -c "import json,sys; d=json.loads(open('$O/${TAG}_${c}_p$p.json').read().strip().splitlines()[-1]); print('$c', $p, d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done > $O/${TAG}_summary.txt
