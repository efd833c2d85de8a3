timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s10_pytest.log 2>&1; echo pytest=$?
bash tools/ab_run.sh s10 paper_1504_03151_b200/libb200rt_base.so paper_1504_03151_b200/libb200rt.so
python tools/depth_profile.py C4 8 > gpurun_out/s10_depth8.log 2>&1
