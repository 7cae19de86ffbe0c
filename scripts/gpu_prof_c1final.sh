mkdir -p gpurun_out/prof
python scripts/prof_missing.py c1 3 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_elementwise -s 3 -c 1 \
   -o gpurun_out/prof/r02_c1_float52_stoch_2p24_warpcta python scripts/prof_missing.py c1 5 > gpurun_out/prof/c1f.log 2>&1
ncu -i gpurun_out/prof/r02_c1_float52_stoch_2p24_warpcta.ncu-rep --page raw --csv > gpurun_out/prof/r02_c1_float52_stoch_2p24_warpcta.raw.csv 2>/dev/null
rm -f gpurun_out/prof/*.ncu-rep; tail -1 gpurun_out/prof/c1f.log
python scripts/ncu_summary.py gpurun_out/prof/r02_c1_float52_stoch_2p24_warpcta.raw.csv
