# ncu --set full captures of the kernel families without a committed raw capture
# (VERDICT r01 missing #6).  Each: plain run first (must exit 0), then one capture.
mkdir -p gpurun_out/prof
M="gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_elapsed.avg,dram__bytes_read.sum,dram__bytes_write.sum"
cap() {  # name kernel-regex skip args...
  local name=$1 k=$2 s=$3; shift 3
  timeout 300 python scripts/prof_missing.py "$@" > gpurun_out/prof/${name}.plain.txt 2>&1 || { echo "$name plain FAILED"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/prof/${name} python scripts/prof_missing.py "$@" > gpurun_out/prof/${name}.ncu.log 2>&1
  ncu -i gpurun_out/prof/${name}.ncu-rep --page raw --csv > gpurun_out/prof/${name}.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/${name}.ncu-rep --page details --csv > gpurun_out/prof/${name}.details.csv 2>/dev/null
  rm -f gpurun_out/prof/${name}.ncu-rep; echo "$name done"
}
cap c1_float52_stoch_2p24 k_elementwise 2 c1 4
cap c1log_float52_stoch_2p24 k_elementwise 2 c1log 4
cap qgemm_general_f52_stoch_2048 k_qgemm_general 1 general 2
cap seg_reduce_whole_2p28 k_seg_reduce 1 seg 2
cap seg_apply_whole_2p28 k_seg_apply 1 seg 2
cap col_reduce_dim1_2p22x64 k_col_reduce 1 col 2
cap col_apply_dim1_2p22x64 k_col_apply 1 col 2
cap group_block_rows_r50w k_group_block_rows 1 group 2
cap group_elementwise_r50w k_group_elementwise 1 group 2
cap encode8_fixed84 k_encode8 2 encode8 2
ls -la gpurun_out/prof
