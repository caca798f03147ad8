# GEMM library variants A/B at the bench shape (stage times of 20 layer
# steps, interleaved): GEMM_VARIANTS="pf8 pf16" bash tools/gemm_ab.sh
for rep in 1 2 3; do
  for v in default ${GEMM_VARIANTS}; do
    if [ $v = default ]; then r=$(python tools/band_sweep.py 20 24 | tail -1); else r=$(MOE_B200_LIB=paper_2508_07329_b200/lib/variants/libmoe_b200_$v.so python tools/band_sweep.py 20 24 | tail -1); fi
    echo "{\"lib\": \"$v\", \"stages\": $r}"
  done
done
