# ncu launch list + full capture of one C5 step (18 kernels), summarised on the box
O=gpurun_out; TAG=${1:-r1f}
KRE='regex:enc_|sif_(parse|dcrc|scatter|dfinal)'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 36 --csv --log-file $O/${TAG}_launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --depth 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none -k "$KRE" -s 18 -c 18 -o $O/${TAG}_full_c5 python bench.py --config c5 --steps 1 --warmup 3 --depth 1 --no-cpu-baseline > /dev/null 2>&1
python tools/make_profiles.py ${TAG} c5:$O/${TAG}_full_c5.ncu-rep > $O/${TAG}_c5prof.log 2>&1
mkdir -p $O/profiles && cp profiles/${TAG}_c5_ncu.txt profiles/ncu_traffic.json $O/profiles/ 2>/dev/null
rm -f $O/${TAG}_full_c5.ncu-rep
