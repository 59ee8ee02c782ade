#!/bin/bash
# Refresh the measurement records under profiles/ on the B200 box.
#   bash tools/refresh_profiles.sh measure   # bench (both arms), config sweep, API overhead, CG example
#   bash tools/refresh_profiles.sh ncu       # bench launch list + ncu --set full summaries of the hot kernels
#   bash tools/refresh_profiles.sh reduce    # round 2: config-3 floors vs product, sweeps, launch floor, group skew
#   bash tools/refresh_profiles.sh all       # everything
# Outputs in gpurun_out/refresh/ (small files only: .ncu-rep files stay in /tmp
# on the box and are summarised there by tools/ncu_summary.py).
set -u
O=gpurun_out/refresh
R=/tmp/salt_reps
mkdir -p $O $R
export NCU=/usr/local/cuda/bin/ncu
T() { timeout "$@"; }
MODE=${1:-measure}
if [ $MODE = measure ] || [ $MODE = all ]; then
  T 900 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?" >> $O/status
  T 600 python bench.py --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/status
  T 1500 python tools/config_sweep.py --out $O/configs.jsonl > $O/configs.log 2>&1; echo "sweep rc=$?" >> $O/status
  T 300 python tools/api_overhead.py > $O/api_overhead.json 2> $O/api.err; echo "api rc=$?" >> $O/status
  T 300 python examples/cg_poisson1d.py --n 1048576 --iters 300 > $O/cg.txt 2>&1; echo "cg rc=$?" >> $O/status
fi
if [ $MODE = ncu ] || [ $MODE = all ]; then
  # launch list of the bench command (cold-cache, serialised; shares only)
  T 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 20 --warmup 3 > $O/bench_ncu.log 2>&1; echo "ncu-launches rc=$?" >> $O/status
  python tools/ncu_summary.py --launches $O/bench_launches.csv --out $O/bench_launches > /dev/null 2>&1
  declare -A BYTES=([t2]=$((32 << 28)) [dot64]=$((16 << 28)) [nrm2_64]=$((8 << 28)) [nrm2_32]=$((4 << 28))
                    [dot32]=$((8 << 28)) [etree32]=$((20 << 30)) [axpydot]=$((32 << 28))
                    [cgupdate]=$((48 << 28)) [daxpy20]=$((24 << 20)) [nrm2_64_mid]=$((8 << 24))
                    [dot64_mid]=$((16 << 24)))
  for c in t2 dot64 nrm2_64 nrm2_32 dot32 etree32 axpydot cgupdate daxpy20 nrm2_64_mid dot64_mid; do
    T 600 python tools/profile_target.py --case $c > $O/pt_$c.log 2>&1 || { echo "target $c failed" >> $O/status; continue; }
    T 900 $NCU --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 \
      -f -o $R/prof_$c python tools/profile_target.py --case $c > $O/ncu_$c.log 2>&1
    echo "ncu $c rc=$?" >> $O/status
    python tools/ncu_summary.py --rep $R/prof_$c.ncu-rep --bytes ${BYTES[$c]} --out $O/ncu_$c \
      --note "ncu --set full of tools/profile_target.py --case $c (one launch after 3 warm-ups)" > /dev/null 2>> $O/status
  done
fi
if [ $MODE = reduce ] || [ $MODE = all ]; then
  # round 2: config 3 product vs bare-read floors in one process (PROBE_SET=final), product sweeps
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -lineinfo -DWITH_SALT -o tools/c3_probe_bin \
    tools/c3_probe.cu -Lpaper_1109_1264_b200 -lsalt -Xlinker -rpath -Xlinker '$ORIGIN/../paper_1109_1264_b200' > $O/c3_nvcc.log 2>&1
  PROBE_SET=final PROBE_LG_LO=20 PROBE_LG_HI=28 T 900 tools/c3_probe_bin 15 > $O/c3_final.txt 2>&1; echo "c3 rc=$?" >> $O/status
  T 600 python tools/reduce_sweep.py > $O/reduce_sweep.jsonl 2> $O/reduce_sweep.err; echo "rsweep rc=$?" >> $O/status
  T 300 python tools/launch_floor_probe.py > $O/launch_floor.json 2> $O/launch_floor.err; echo "floor rc=$?" >> $O/status
  T 300 python tools/group_issue_probe.py > $O/group_issue.json 2> $O/group_issue.err; echo "group rc=$?" >> $O/status
fi

