#!/bin/bash
# Round-2 profiles (run from the repo root under gpurun): the launch list of
# the default bench command, and `ncu --set full` captures of the kernels this
# round added or changed.  Outputs go to gpurun_out/prof2/.
set -u
mkdir -p gpurun_out/prof2
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof2/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof2/launches_config3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof2/ncu_launches.log 2>&1
full() {  # name, kernel regex, command...  (SKIP=n: skip the first n matching launches)
  local name=$1 kre=$2; shift 2
  "$@" > gpurun_out/prof2/$name.plain.log 2>&1 || { echo "$name: command failed"; return; }
  ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip ${SKIP:-0} -c 1 \
      -o gpurun_out/prof2/$name "$@" > gpurun_out/prof2/$name.log 2>&1
}
SKIP=1 full resid_k64 resid_gram_kernel python tools/diag/resid_probe.py --m 32000000 --k 64 --reps 1
SKIP=1 full factor_k256 factor_kernel python tools/kernel_probe.py --only factor --fk 256 --reps 1
full gram_k256 gram_pairs_kernel python tools/kernel_probe.py --only gram --m 2000000 --k 256 --reps 1
full trmm_k256 gemm_kernel python tools/kernel_probe.py --only apply --m 2000000 --k 256 --reps 1
ls -la gpurun_out/prof2
