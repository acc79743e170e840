O=gpurun_out; TAG=bk
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 400 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:enc_token|sif_dec_small' -c 20 --csv --log-file $O/${TAG}_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
timeout 900 $CS --tool memcheck $PT tests/test_gpu_parity.py tests/test_gpu_workloads.py::test_c3_every_token_matches_reference > $O/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/${TAG}_memcheck.log
timeout 900 $CS --tool racecheck --racecheck-report all $PT tests/test_gpu_parity.py > $O/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/${TAG}_racecheck.log
timeout 600 $CS --tool synccheck $PT tests/test_gpu_parity.py > $O/${TAG}_synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/${TAG}_synccheck.log
for t in memcheck racecheck synccheck; do echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_$t.log | tail -3; done > $O/${TAG}_summary.txt
