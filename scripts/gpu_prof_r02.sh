# ncu --set full captures of this round's new kernels (each: plain run first, then one capture)
mkdir -p gpurun_out/prof2
cap() {  # name kernel-regex skip script args...
  local name=$1 k=$2 s=$3; shift 3
  timeout 300 python "$@" > gpurun_out/prof2/${name}.plain.txt 2>&1 || { echo "$name plain FAILED"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/prof2/${name} python "$@" > gpurun_out/prof2/${name}.ncu.log 2>&1
  ncu -i gpurun_out/prof2/${name}.ncu-rep --page raw --csv > gpurun_out/prof2/${name}.raw.csv 2>/dev/null
  rm -f gpurun_out/prof2/${name}.ncu-rep; echo "$name done"
}
cap r02_chunk_act_sr_256x802816 k_block_chunks 2 scripts/prof_kernel.py acts 0 4
cap r02_qgemm_bits_f87_stoch_2048 k_qgemm_bits 1 scripts/prof_missing.py bits 2
