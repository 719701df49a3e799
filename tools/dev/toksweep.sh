#!/bin/bash
# K5 / K8 build variants (token loads in flight x min blocks per SM), each a
# separate libdpcuda.so under build/var_*, timed through bench.py.
for d in build/var_*; do
  for c in cfg4 cfg4r cfg4b; do
    DP_LIB_PATH=$d/libdpcuda.so python bench.py --config $c > gpurun_out/sw.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/sw.log').readlines()[-1]);print('$d $c', round(d['value']/1e6,1), d['roofline']['frac'], d['roofline']['avg_launch_us'])"
  done
done
