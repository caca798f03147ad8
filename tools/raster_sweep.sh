# GEMM raster / L2-policy sweep at the bench shape: ncu DRAM bytes and time
# of the two grouped GEMM launches per (band MB, policy) setting.
for cfg in 24:0 96:0 96:8 96:2 6:0 6:2 3:0 3:8; do
  mb=${cfg%%:*}; pol=${cfg##*:}
  MOE_B200_GEMM_L2POL=$pol MOE_B200_BAND_ONE=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_i8_tc --csv --log-file gpurun_out/raster_${mb}_${pol}.csv \
    python tools/band_sweep.py 1 > /dev/null 2>&1
done
