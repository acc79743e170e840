for p in 1 2 4; do timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --parts $p > gpurun_out/parts_c3_$p.json 2>/dev/null; done
for p in 8 16; do timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --parts $p > gpurun_out/parts_c2_$p.json 2>/dev/null; done
