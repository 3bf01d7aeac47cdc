#!/bin/bash
# Re-captures every committed ncu artefact for the current code (GPU box, one GPU):
#   traffic per precision (capture_traffic.sh), the bench launch list, full captures of the engine
#   at p=2 and p=4.  Each ncu command runs only after the same command exited 0 without ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/capture_traffic.sh
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-prefill --no-fp16"
$B > gpurun_out/bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"engine_kernel|sched_step" -c 200 --csv \
      --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch.log 2>&1
for p in 2 4; do
  python tools/profile_token.py $p engine > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 3 -c 1 \
      -o gpurun_out/prof_engine_p$p -f python tools/profile_token.py $p engine > /dev/null 2>&1
done
echo refresh done
