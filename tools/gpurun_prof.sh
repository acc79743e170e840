# usage: bash tools/gpurun_prof.sh TAG "cfg:kernelregex:skip ..." -- one ncu --set full capture per entry, summaries
TAG=${1:-p}; shift
O=gpurun_out
for spec in $1; do
  c=${spec%%:*}; rest=${spec#*:}; k=${rest%%:*}; s=${rest##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s $s -c 1 -o $O/${TAG}_${c}_${k} python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --depth 1 > /dev/null 2>&1
  python tools/ncu_summary.py $O/${TAG}_${c}_${k}.ncu-rep > $O/${TAG}_${c}_${k}_summary.txt 2>&1
  python tools/ncu_hot.py $O/${TAG}_${c}_${k}.ncu-rep 40 > $O/${TAG}_${c}_${k}_hot.txt 2>&1
done
