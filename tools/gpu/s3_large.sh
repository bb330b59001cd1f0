timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_edges.py -x -q 2>&1 | tail -5 > gpurun_out/s3_large_test.txt
python tools/c5_split.py 1000000 > gpurun_out/s3_c5_time.txt 2>&1
for r in "2,2" "2,3" "3,2" "1,2" "2,1"; do echo "rep $r: $(QLM_LARGE_REP=$r python tools/c5_split.py 1000000 2>&1 | tail -1)" >> gpurun_out/s3_c5_time.txt; done
cat gpurun_out/s3_large_test.txt gpurun_out/s3_c5_time.txt
