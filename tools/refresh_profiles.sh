#!/bin/bash
# One GPU call that refreshes every measurement record under profiles/:
#   config sweep, bench (both arms), bench launch list, ncu --set full of the
#   hot kernels, API overhead, PCIe ceiling, CPU reference engines.
# Run on the B200 box:  bash tools/refresh_profiles.sh  (outputs in gpurun_out/refresh/)
set -u
O=gpurun_out/refresh
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
T() { timeout "$@"; }
T 900 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?" >> $O/status
T 600 python bench.py --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/status
T 1500 python tools/config_sweep.py --out $O/configs.jsonl > $O/configs.log 2>&1; echo "sweep rc=$?" >> $O/status
T 300 python tools/api_overhead.py > $O/api_overhead.json 2> $O/api.err; echo "api rc=$?" >> $O/status
T 300 python examples/cg_poisson1d.py --n 1048576 --iters 300 > $O/cg.txt 2>&1; echo "cg rc=$?" >> $O/status
# launch list of the bench command (cold-cache, serialised; shares only)
T 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 20 --warmup 3 > $O/bench_ncu.log 2>&1; echo "ncu-launches rc=$?" >> $O/status
for c in t2 dot64 nrm2_64 nrm2_32 dot32 etree32 axpydot cgupdate daxpy20; do
  T 600 python tools/profile_target.py --case $c > $O/pt_$c.log 2>&1 || { echo "target $c failed" >> $O/status; continue; }
  T 900 $NCU --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 \
    -o $O/prof_$c python tools/profile_target.py --case $c > $O/ncu_$c.log 2>&1
  echo "ncu $c rc=$?" >> $O/status
done
