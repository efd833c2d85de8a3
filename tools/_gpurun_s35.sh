timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -x -q > gpurun_out/s35_pytest.log 2>&1; echo pytest=$?
B200RT_LIB=$PWD/paper_1504_03151_b200/libb200rt_lt4.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -x -q > gpurun_out/s35_pytest_lt4.log 2>&1; echo pytest4=$?
bash tools/ab_run.sh s35 paper_1504_03151_b200/libb200rt_prev.so paper_1504_03151_b200/libb200rt.so paper_1504_03151_b200/libb200rt_lt3.so paper_1504_03151_b200/libb200rt_lt4.so
