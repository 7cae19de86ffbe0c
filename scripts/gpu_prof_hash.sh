# ncu captures after the shared >> 30 hash word (round 2, late)
mkdir -p gpurun_out/prof
python scripts/prof_kernel.py c1 24 5 && python scripts/prof_kernel.py acts 0 3 && python scripts/prof_kernel.py c2 30 3 || exit 1
cap() {  # name kernel-regex cfg nlog reps skip
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s $6 -c 1 \
     -o gpurun_out/prof/$1 python scripts/prof_kernel.py $3 $4 $5 > gpurun_out/prof/$1.log 2>&1
  ncu -i gpurun_out/prof/$1.ncu-rep --page raw --csv > gpurun_out/prof/$1.raw.csv 2>/dev/null
  rm -f gpurun_out/prof/$1.ncu-rep; tail -1 gpurun_out/prof/$1.log
}
cap r02_c1_float52_stoch_2p24_hash30 k_elementwise c1 24 5 3
cap r02_chunk_act_sr_256x802816_hash30 k_block_chunks acts 0 3 1
cap r02_c2_fixed84_stoch_2p30_hash30 k_elementwise c2 30 3 1
python scripts/ncu_summary.py gpurun_out/prof/*.raw.csv
