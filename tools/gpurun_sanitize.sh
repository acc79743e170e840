# usage: bash tools/gpurun_sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck / initcheck
# over the GPU parity suite, checking only this library's kernels (mangled names contain "sif").
TAG=${1:-san}
O=gpurun_out
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
SEL="tests/test_gpu_parity.py tests/test_gpu_ref_api.py tests/test_gpu_random.py::test_path_boundaries_match_oracle tests/test_gpu_random.py::test_multi_kernel_select_path_matches_oracle tests/test_gpu_random.py::test_ms_cut_at_last_element_of_large_tie_group tests/test_gpu_random.py::test_per_if_back_end_matches_oracle tests/test_gpu_random.py::test_stream_ring_tails_match_oracle tests/test_gpu_workloads.py::test_batch_pipeline_refilled_inputs tests/test_gpu_workloads.py::test_c3_every_token_matches_reference"
SMALL="tests/test_gpu_parity.py::test_encode_decode_golden tests/test_gpu_parity.py::test_structural_streams tests/test_gpu_parity.py::test_many_blocks_match_reference"
timeout 1500 $CS --tool memcheck $PT tests > $O/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/${TAG}_memcheck.log
timeout 1200 $CS --tool racecheck --racecheck-report all $PT $SEL > $O/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/${TAG}_racecheck.log
timeout 600 $CS --tool synccheck $PT $SEL > $O/${TAG}_synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/${TAG}_synccheck.log
timeout 900 $CS --tool initcheck $PT $SMALL > $O/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?" >> $O/${TAG}_initcheck.log
for t in memcheck racecheck synccheck initcheck; do echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_$t.log | tail -4; done > $O/${TAG}_summary.txt
