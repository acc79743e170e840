# usage: bash tools/gpurun_san_wide.sh [TAG] -- GPU tests, then memcheck / racecheck / synccheck over the many-block (> 32 effective blocks) paths
O=gpurun_out; TAG=${1:-sanw}
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
SEL="tests/test_gpu_parity.py::test_many_blocks_match_reference tests/test_gpu_random.py::test_per_if_back_end_matches_oracle tests/test_gpu_random.py::test_random_sweep_matches_oracle"
for t in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $t $PT $SEL > $O/${TAG}_$t.log 2>&1; echo "$t rc=$?" >> $O/${TAG}_$t.log
done
for t in memcheck racecheck synccheck; do echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_$t.log | tail -4; done > $O/${TAG}_summary.txt
