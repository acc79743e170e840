O=gpurun_out
for t in 131072 65536 32768; do SIF_BIG_NCAND=$t timeout 600 python bench.py --config c5 --steps 5 --warmup 2 --no-cpu-baseline > $O/big_c5_$t.json 2> $O/big_c5_$t.err; done
for t in 131072 16384; do SIF_BIG_NCAND=$t timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/big_c2_$t.json 2> $O/big_c2_$t.err; done
