mkdir -p gpurun_out/full
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full/pytest.txt 2>&1; tail -5 gpurun_out/full/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1; cat gpurun_out/full/smoke.txt
timeout 600 python bench.py > gpurun_out/full/bench.json 2> gpurun_out/full/bench.err; cat gpurun_out/full/bench.json
