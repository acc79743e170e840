# Run the REFERENCE's own codec/ATKF tests (tests/test_codec.py, tests/test_atkf.py) against
# the `slicer`-named shim over the GPU codec.  Step 1 (build container, where /root/reference
# exists): copy the two test files into the git-ignored baseline/_ref_tests/.  Step 2 (GPU
# box via gpurun): run them with the shim first on sys.path.
#   bash tools/run_reference_tests.sh copy        # here
#   gpurun -- 'bash tools/run_reference_tests.sh run > gpurun_out/reftests.log 2>&1'
set -e
D=baseline/_ref_tests
if [ "$1" = "copy" ]; then
  mkdir -p $D && cp /root/reference/pkg/tests/test_codec.py /root/reference/pkg/tests/test_atkf.py $D/
  exit 0
fi
cd $D
PYTHONPATH=$GRAFT_REPO_ROOT/paper_2511_11608_b200/compat:$GRAFT_REPO_ROOT python -c "import slicer; print('slicer ->', slicer.__file__)"
PYTHONPATH=$GRAFT_REPO_ROOT/paper_2511_11608_b200/compat:$GRAFT_REPO_ROOT python -m pytest -q -p no:cacheprovider test_codec.py test_atkf.py --rootdir=. 2>&1
