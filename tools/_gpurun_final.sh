# Final round check on one GPU: build + smoke, GPU tests, the default bench line.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo bench=$?
