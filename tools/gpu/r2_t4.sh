timeout 600 python -m pytest tests/test_gpu_comm.py -q -x 2>&1 | tail -15 > gpurun_out/comm.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 >> gpurun_out/comm.txt
cat gpurun_out/comm.txt
