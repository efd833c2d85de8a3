timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s15_pytest.log 2>&1; echo pytest=$?
timeout 300 python tools/depth_profile.py C4 8 > gpurun_out/s15_depth8.log 2>&1
timeout 300 python tools/graph_probe.py C4 > gpurun_out/s15_probe.log 2>&1
