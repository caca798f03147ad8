# K1 on h: bulk-ring kernel (default) vs the register row kernel, interleaved
for rep in 1 2 3; do
  python tools/k1x_ab.py 30
  MOE_B200_K1_CFG=0 python tools/k1x_ab.py 30 | sed 's/"lib": "default"/"lib": "warp_cfg0"/'
done
