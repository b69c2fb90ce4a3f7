for cfg in "QLRT_CL2=0" "QLRT_CL2=1" "QLRT_OVERLAP_BWD=1 QLRT_CL2=0" "QLRT_OVERLAP_BWD=1 QLRT_CL2=2" "QLRT_OVERLAP_BWD=1 QLRT_CL2=3"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/bench_c3.py 7b --layers 8 --steps 10 2>&1 | tail -1 | cut -c60-140
done
