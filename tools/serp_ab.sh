# A/B of the grouped GEMM's serpentine k order (MOE_B200_GEMM_SERP, default
# on) at the bench shape: stage times of 20 layer steps, interleaved
for rep in 1 2 3; do
  for v in 0 1; do
    r=$(MOE_B200_GEMM_SERP=$v python tools/band_sweep.py 20 24 | tail -1)
    echo "serp=$v $r"
  done
done
