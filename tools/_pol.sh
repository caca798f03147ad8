for b in 24 48 64 128; do
  echo "== band $b MB"
  for i in 1 2; do MOE_B200_BAND_MB=$b timeout 300 python tools/gemm_bench.py 2>&1 | grep -E "gemm2"; done
  MOE_B200_BAND_MB=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_i8_tc -s 57 -c 10 --csv python tools/gemm_bench.py 2>/dev/null | python tools/ncu_pick.py
done
