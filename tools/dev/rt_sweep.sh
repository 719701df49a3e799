# dev: A/B the ragged-batch kernel's block shape (cfg4r); variant .so files
# built with make EXTRA_NVCCFLAGS="-DDP_TOK_RAGGED_THREADS=T -DDP_TOK_RAGGED_TILE=R"
for r in 1 2 3 4; do
for v in ${VARIANTS:-default var_rt128_64}; do
  if [ $v = default ]; then unset DP_LIB_PATH; else export DP_LIB_PATH=$PWD/build/$v/libdpcuda.so; fi
  printf "%s " $v; python bench.py --config ${CFG:-cfg4r} --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])"
done; done
