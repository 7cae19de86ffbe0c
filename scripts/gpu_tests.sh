mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.txt
build/dropin/lpsim_acceptance_b200 > gpurun_out/acceptance.txt 2>&1; echo rc=$? >> gpurun_out/acceptance.txt
build/dropin/lpsim_tests_b200 > gpurun_out/dropin_tests.txt 2>&1; echo rc=$? >> gpurun_out/dropin_tests.txt
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/acceptance.txt; tail -4 gpurun_out/dropin_tests.txt
