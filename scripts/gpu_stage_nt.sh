# criterion 7 host-call timing (scripts/host_crit7.cpp: the acceptance
# harness restated against the C ABI) and the drop-in acceptance binary
mkdir -p gpurun_out/nt
g++ -O2 -std=c++17 scripts/host_crit7.cpp -Iinclude -Lpaper_1910_04540_b200/lib -llpq \
    -Wl,-rpath,$PWD/paper_1910_04540_b200/lib -o gpurun_out/nt/crit7
for r in 1 2; do
  timeout 300 gpurun_out/nt/crit7 | grep "round [12]"
  timeout 600 build/dropin/lpsim_acceptance_b200 2>&1 | grep "criterion 7"
done
python scripts/pcie_parts_probe.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_quantize.py tests/test_gpu_vs_reference_lib.py tests/test_gpu_dropin.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
