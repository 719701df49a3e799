# dev: K5 ragged flat-span variant -- parity tests, then interleaved A/B on cfg4r
export DP_LIB_PATH=$PWD/build/var_flat16/libdpcuda.so
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ragged or cfg4r or token" 2>&1 | tail -2
unset DP_LIB_PATH
VARIANTS="default var_flat16 var_flat8 var_flat32" CFG=cfg4r bash tools/dev/rt_sweep.sh
