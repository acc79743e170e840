O=gpurun_out
for d in 3 4 6; do timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --depth $d > $O/depth_c2_$d.json 2>/dev/null; done
for d in 2 4 6; do timeout 400 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline --depth $d > $O/depth_c4_$d.json 2>/dev/null; done
for d in 4 8; do timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --depth $d > $O/depth_c3_$d.json 2>/dev/null; done
