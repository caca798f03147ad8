# A/B of K1 variants, interleaved (thermal drift hits all variants alike)
for rep in 1 2 3; do
  for v in default ${K1_VARIANTS:-nopf}; do
    if [ $v = default ]; then python tools/k1x_ab.py 30; else MOE_B200_LIB=paper_2508_07329_b200/lib/variants/libmoe_b200_$v.so python tools/k1x_ab.py 30; fi
  done
done
