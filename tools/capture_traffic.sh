#!/bin/bash
# ncu DRAM traffic of one engine launch (7B linear stack token) per precision -> gpurun_out/traffic_p*.csv
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for p in 4 3 2; do
  python tools/profile_token.py $p engine > gpurun_out/plain_p$p.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:engine_kernel -s 3 -c 1 --csv --log-file gpurun_out/traffic_p$p.csv \
      python tools/profile_token.py $p engine > /dev/null 2>&1
done
