for cfg in 1:0 1:2 1:8 2:2; do
  mb=${cfg%%:*}; pol=${cfg##*:}
  MOE_B200_GEMM_L2POL=$pol MOE_B200_BAND_ONE=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gemm_i8_tc --csv --log-file gpurun_out/raster_${mb}_${pol}.csv \
    python tools/band_sweep.py 1 > /dev/null 2>&1
done
