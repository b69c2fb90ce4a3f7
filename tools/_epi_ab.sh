L=paper_2305_14314_b200/_lib
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or linear or llama or qlinear" 2>&1 | tail -5
for s in 4096x11008 8192x22016; do
 for rep in 1 2; do
  for v in libqlrt_b200 libqlrt_old; do
   echo -n "$v "; QLRT_LIB_PATH=$L/$v.so timeout 120 python tools/ab.py QLRT_TMAOUT=1 QLRT_TMAOUT=0 --shape $s --rounds 3
  done
 done
done
for v in libqlrt_b200 libqlrt_old; do echo $v; QLRT_LIB_PATH=$L/$v.so timeout 300 python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"; done
