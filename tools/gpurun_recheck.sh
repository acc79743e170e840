O=gpurun_out; TAG=san2f
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
timeout 900 $CS --tool racecheck --racecheck-report all $PT tests/test_gpu_parity.py > $O/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/${TAG}_racecheck.log
grep -E "RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_racecheck.log | tail -3 > $O/${TAG}_summary.txt
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
SIF_PLAN_CACHE=1 timeout 600 python bench.py --gpus 2 --config c2 --steps 5 --warmup 3 --no-cpu-baseline > $O/dry2_c2.json 2> $O/dry2_c2.err
timeout 900 python bench.py --gpus 2 --config c5 --steps 3 --warmup 3 --no-cpu-baseline > $O/dry2_c5.json 2> $O/dry2_c5.err
