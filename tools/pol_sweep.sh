python -m pytest tests/test_gpu_kernels.py tests/test_gpu_bench_parity.py tests/test_gpu_moe.py -m gpu -x -q > gpurun_out/pytest3.log 2>&1; echo pytest_rc=$?
for rep in 1 2 3; do for pol in 0 8 4 5 2 9; do echo "pol=$pol rep=$rep $(MOE_B200_GEMM_L2POL=$pol python tools/band_sweep.py 20 24 2>&1 | tail -1)" >> gpurun_out/pol.log; done; done
for pol in 0 8 5 2; do MOE_B200_GEMM_L2POL=$pol MOE_B200_BAND_ONE=24 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_i8_tc|act_quant" --csv --log-file gpurun_out/pol_ncu_$pol.csv python tools/band_sweep.py 1 > /dev/null 2>&1; done
tail -2 gpurun_out/pytest3.log
