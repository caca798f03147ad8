# Whole-layer bench of the in-tree library against another build, interleaved
# (thermal drift hits both alike):  VARIANT=path/to/libmoe_b200_x.so bash tools/lib_ab.sh
for rep in 1 2 3; do
  for v in default "${VARIANT:?set VARIANT to a library path}"; do
    if [ "$v" = default ]; then lib=""; else lib="$v"; fi
    r=$(MOE_B200_LIB=$lib python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
    echo "$(basename "$v") $r"
  done
done
