O=gpurun_out; TAG=san2d
timeout 900 python -m pytest tests -x -q -m gpu > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
CS="compute-sanitizer --kernel-name kns=sif --print-limit 50 --error-exitcode 99"
PT="python -m pytest -x -q -m gpu -p no:cacheprovider"
SEL="tests/test_gpu_parity.py tests/test_gpu_ref_api.py tests/test_gpu_random.py::test_path_boundaries_match_oracle tests/test_gpu_random.py::test_multi_kernel_select_path_matches_oracle tests/test_gpu_random.py::test_ms_cut_at_last_element_of_large_tie_group tests/test_gpu_random.py::test_per_if_back_end_matches_oracle tests/test_gpu_random.py::test_stream_ring_tails_match_oracle tests/test_gpu_workloads.py::test_batch_pipeline_refilled_inputs tests/test_gpu_workloads.py::test_c3_every_token_matches_reference"
SMALL="tests/test_gpu_parity.py::test_encode_decode_golden tests/test_gpu_parity.py::test_structural_streams tests/test_gpu_parity.py::test_many_blocks_match_reference tests/test_gpu_parity.py::test_corrupt_streams_error_classes"
timeout 1200 $CS --tool racecheck --racecheck-report all $PT $SEL > $O/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/${TAG}_racecheck.log
timeout 900 $CS --tool initcheck $PT $SMALL > $O/${TAG}_initcheck.log 2>&1; echo "initcheck rc=$?" >> $O/${TAG}_initcheck.log
for t in racecheck initcheck; do echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $O/${TAG}_$t.log | tail -4; done > $O/${TAG}_summary.txt
bash tools/gpurun_prof.sh p2c "c2:enc_stream:3"
