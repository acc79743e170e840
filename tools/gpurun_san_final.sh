# usage: bash tools/gpurun_san_final.sh [TAG] -- memcheck over the parity suite and racecheck / synccheck over the
# single-IF graph-replay, many-block and multi-kernel select tests on the final code
O=gpurun_out; TAG=${1:-sanf}
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
SEL="tests/test_gpu_parity.py::test_graph_replayed_single_if_calls tests/test_gpu_parity.py::test_cached_calls_follow_routing_changes tests/test_gpu_parity.py::test_many_blocks_match_reference tests/test_gpu_random.py::test_multi_kernel_select_path_matches_oracle"
timeout 1500 $CS --tool memcheck $PT tests/test_gpu_parity.py tests/test_gpu_random.py > $O/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/${TAG}_memcheck.log
for t in racecheck synccheck; do
  timeout 1500 $CS --tool $t $PT $SEL > $O/${TAG}_$t.log 2>&1; echo "$t rc=$?" >> $O/${TAG}_$t.log
done
for t in memcheck racecheck synccheck; do echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_$t.log | tail -4; done > $O/${TAG}_summary.txt
