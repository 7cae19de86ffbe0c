# One GPU session: smoke, tests (optional), benches, ncu captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke=$? >> gpurun_out/smoke.txt
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.txt
fi
for c in c2 c3 c3s c1 c1n c1big c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != c2 ] && echo --no-e2e --no-cpu ) > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 300 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
if [ "${NCU:-1}" = 1 ]; then
  python scripts/prof_kernel.py c2 30 2 > gpurun_out/prof_plain_c2.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_elementwise -s 1 -c 1 \
      -o gpurun_out/prof_c2 python scripts/prof_kernel.py c2 30 2 > gpurun_out/ncu_c2.log 2>&1
  python scripts/prof_kernel.py c3 28 2 > gpurun_out/prof_plain_c3.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_block_rows -s 1 -c 1 \
      -o gpurun_out/prof_c3 python scripts/prof_kernel.py c3 28 2 > gpurun_out/ncu_c3.log 2>&1
  python scripts/prof_gemm.py 4096 2 > gpurun_out/prof_plain_gemm.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_qgemm_bf16 -s 1 -c 1 \
      -o gpurun_out/prof_gemm python scripts/prof_gemm.py 4096 2 > gpurun_out/ncu_gemm.log 2>&1
  python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launches.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.txt 2>/dev/null
for c in c2 c3 c3s c1 c1n c1big c5 c4; do python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); r=d['roofline']
print('$c', d['value'], d['unit'], 'frac', r['frac'], 'e2e', (d.get('e2e') or {}).get('value'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; done
