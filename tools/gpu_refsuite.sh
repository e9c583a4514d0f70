# the reference's own unit suite and acceptance criteria linked against the GPU backend
mkdir -p gpurun_out
cd paper_2407_13055_b200/_lib/ref_gpu
( time timeout 900 ./ref_unit_tests_gpu ) > $GRAFT_REPO_ROOT/gpurun_out/ref_unit_gpu.txt 2>&1; echo "unit rc=$?"
grep -E "FAIL|test cases failed" $GRAFT_REPO_ROOT/gpurun_out/ref_unit_gpu.txt | head -40
( time timeout 1500 ./acceptance_gpu /nonexistent-cli ) > $GRAFT_REPO_ROOT/gpurun_out/ref_accept_gpu.txt 2>&1; echo "accept rc=$?"
cat $GRAFT_REPO_ROOT/gpurun_out/ref_accept_gpu.txt | tail -15
