# round-end check: the GPU suite, smoke(), the driver's default bench line and its launch list
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest.txt 2>&1; tail -3 gpurun_out/final/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; cat gpurun_out/final/smoke.txt
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; cat gpurun_out/final/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/final/ncu.log 2>&1
tail -1 gpurun_out/final/ncu.log | cut -c1-200
