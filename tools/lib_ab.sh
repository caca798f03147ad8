for rep in 1 2 3; do
  for v in default old; do
    if [ $v = default ]; then lib=""; else lib=paper_2508_07329_b200/lib/variants/libmoe_b200_old.so; fi
    r=$(MOE_B200_LIB=$lib python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4))")
    echo "$v $r"
  done
done
