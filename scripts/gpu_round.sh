# One GPU session: tests, smoke, benches, then an ncu capture of the C2 kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke=$? >> gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.txt
for c in c2 c3 c1 c1n; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != c2 ] && echo --no-e2e --no-cpu ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
if [ "${NCU:-1}" = 1 ]; then
  python scripts/prof_kernel.py c2 28 3 > gpurun_out/prof_plain.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_elementwise -s 1 -c 1 \
      -o gpurun_out/prof_c2 python scripts/prof_kernel.py c2 28 3 > gpurun_out/ncu_c2.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench_*.json
