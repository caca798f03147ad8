# A/B of the serpentine k order in the grouped GEMM (MOE_B200_GEMM_SERP): stage times at the bench shape
for rep in 1 2 3; do
  for v in 0 1; do
    r=$(MOE_B200_GEMM_SERP=$v python tools/band_sweep.py 20 24 | tail -1)
    echo "serp=$v $r"
  done
done
