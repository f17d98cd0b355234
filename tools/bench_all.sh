#!/bin/bash
# Full 1-GPU measurement set for one round tag: every BASELINE config, the reference arm, and the
# ncu launch list of the default bench command.  Usage: bash tools/bench_all.sh r01c
tag=${1:-rXX}
mkdir -p gpurun_out/$tag
for c in 1 2 3 4 5a 5b solve; do
  timeout 900 python bench.py --config $c > gpurun_out/$tag/bench_cfg$c.json 2> gpurun_out/$tag/bench_cfg$c.err
  echo "cfg $c rc=$?"; tail -c 400 gpurun_out/$tag/bench_cfg$c.json
done
timeout 600 python bench.py --impl reference > gpurun_out/$tag/ref_cfg2.json 2> gpurun_out/$tag/ref_cfg2.err
echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/$tag/ncu_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu \
  > gpurun_out/$tag/ncu_launches.log 2>&1
echo "ncu rc=$?"
