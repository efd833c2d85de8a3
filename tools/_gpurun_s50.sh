timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s50_pytest.log 2>&1; echo pytest=$?
bash tools/ab_run.sh s50 paper_1504_03151_b200/libb200rt_prev.so paper_1504_03151_b200/libb200rt.so
