# A/B two library builds on the C3 bench step: LIBS="b200 other" bash tools/ab_c3.sh (libqlrt_<name>.so in _lib/)
L=paper_2305_14314_b200/_lib
for rep in 1 2; do
 for v in ${LIBS:-b200 hint}; do
  echo -n "$v "; QLRT_LIB_PATH=$L/libqlrt_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))"
 done
done
