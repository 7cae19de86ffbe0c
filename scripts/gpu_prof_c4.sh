mkdir -p gpurun_out/prof
python scripts/prof_missing.py exact 2 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_qgemm_bf16<\(bool\)1, \(bool\)0>' -s 1 -c 1 \
   -o gpurun_out/prof/r02_c4_qgemm_exact_4096 python scripts/prof_missing.py exact 2 > gpurun_out/prof/c4.log 2>&1
ncu -i gpurun_out/prof/r02_c4_qgemm_exact_4096.ncu-rep --page raw --csv > gpurun_out/prof/r02_c4_qgemm_exact_4096.raw.csv 2>/dev/null
ncu -i gpurun_out/prof/r02_c4_qgemm_exact_4096.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/r02_c4_qgemm_exact_4096.sass.csv 2>/dev/null
rm -f gpurun_out/prof/r02_c4_qgemm_exact_4096.ncu-rep; tail -1 gpurun_out/prof/c4.log
python scripts/ncu_summary.py gpurun_out/prof/r02_c4_qgemm_exact_4096.raw.csv
