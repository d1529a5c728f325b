#!/bin/bash
# Round-2 (second session) profiles of the band-cluster k x k stage, from the
# repo root under gpurun: the launch list of the default bench command, and
# `ncu --set full` captures of one cluster factor launch (k = 256: plain, and
# the speculative RECOMPUTE launch whose plain attempt breaks down) plus the
# single-CTA path on the same Gramian for comparison.  Outputs: gpurun_out/prof3/.
set -u
mkdir -p gpurun_out/prof3
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof3/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof3/launches_config3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof3/ncu_launches.log 2>&1
full() {  # name, kernel regex, command...  (the 3rd matching launch: after two warm calls)
  local name=$1 kre=$2; shift 2
  "$@" > gpurun_out/prof3/$name.plain.log 2>&1 || { echo "$name: command failed"; return; }
  ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip 2 -c 1 \
      -o gpurun_out/prof3/$name "$@" > gpurun_out/prof3/$name.log 2>&1
}
full factor_cluster_k256_plain 'factor_kernel' python tools/diag/factor_one.py 256 plain spd 1
full factor_cluster_k256_recompute 'factor_kernel' python tools/diag/factor_one.py 256 recompute illcond 1
full factor_single_k256_plain 'factor_kernel' python tools/diag/factor_one.py 256 plain spd 0
full finish_k256 'factor_finish_kernel' python tools/diag/factor_one.py 256 plain spd 1
ls -la gpurun_out/prof3
