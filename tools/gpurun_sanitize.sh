# usage: bash tools/gpurun_sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / initcheck / synccheck
# over the GPU parity suite, checking only this library's kernels (namespace sif::).
TAG=${1:-san}
timeout 300 python tools/phase_prof.py c3 > gpurun_out/${TAG}_phase_c3.txt 2>&1
O=gpurun_out
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
SEL_FAST="tests/test_gpu_parity.py tests/test_gpu_ref_api.py tests/test_gpu_random.py::test_path_boundaries_match_oracle tests/test_gpu_random.py::test_multi_kernel_select_path_matches_oracle tests/test_gpu_random.py::test_ms_cut_at_last_element_of_large_tie_group tests/test_gpu_random.py::test_per_if_back_end_matches_oracle tests/test_gpu_workloads.py::test_batch_pipeline_refilled_inputs"
timeout 2400 $CS --tool memcheck $PT tests > $O/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/${TAG}_memcheck.log
timeout 1500 $CS --tool initcheck $PT $SEL_FAST > $O/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?" >> $O/${TAG}_initcheck.log
timeout 2400 $CS --tool racecheck --racecheck-report all $PT $SEL_FAST > $O/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/${TAG}_racecheck.log
timeout 1500 $CS --tool synccheck $PT $SEL_FAST > $O/${TAG}_synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/${TAG}_synccheck.log
for t in memcheck initcheck racecheck synccheck; do tail -3 $O/${TAG}_$t.log; done
