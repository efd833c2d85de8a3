timeout 600 python -m pytest tests/test_gpu_split.py -x -q > gpurun_out/s41_split.log 2>&1; echo split=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s41_pytest.log 2>&1; echo pytest=$?
bash tools/ab_run.sh s41 paper_1504_03151_b200/libb200rt_prev.so paper_1504_03151_b200/libb200rt.so
