#!/bin/bash
mkdir -p gpurun_out/lat2
for lib in ab/sb.so ab/cur.so ab/start.so; do
  for n in 100 400 1000; do
    MINE_B200_LIB=$PWD/$lib timeout 300 python tools/per_pair_latency.py $n 300 >> gpurun_out/lat2/$(basename $lib .so).jsonl 2>>gpurun_out/lat2/err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi_gpu.py -x -q > gpurun_out/lat2/pytest.log 2>&1
tools/ab_libs.sh gpurun_out/lat2 "0:256:7 2:20000:5 3:2000:3" ab/sb.so ab/cur.so
