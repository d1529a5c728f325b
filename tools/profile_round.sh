#!/bin/bash
# Capture the round's profiles on a GPU box (run from the repo root under gpurun):
#   launch list of the default bench command, and one `ncu --set full` capture
#   per hot kernel.  Outputs go to gpurun_out/prof/.
set -u
mkdir -p gpurun_out/prof
python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/bench_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_config3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_launches.log 2>&1
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/bench_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_config5.csv \
    python bench.py --config 5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof/ncu_launches5.log 2>&1
full() {  # name, kernel regex, command...  (SKIP=n: skip the first n matching launches)
  local name=$1 kre=$2; shift 2
  "$@" > /dev/null 2>&1 || { echo "$name: command failed"; return; }
  ncu --set full --clock-control none --import-source on -k "regex:$kre" --launch-skip ${SKIP:-0} -c 1 \
      -o gpurun_out/prof/$name "$@" \
      > gpurun_out/prof/$name.log 2>&1
}
full gram_k256 gram_pairs_kernel python tools/kernel_probe.py --only gram --m 2000000 --k 256 --reps 1
full trmm_k256 gemm_kernel python tools/kernel_probe.py --only apply --m 2000000 --k 256 --reps 1
full gram_k64 apply_gram_rt_kernel python tools/kernel_probe.py --only gram --m 32000000 --k 64 --reps 1
# kernel_probe --only apply runs one plain Gram (the TRMM-less instance of the same kernel) first
SKIP=1 full fused_k64 apply_gram_rt_kernel python tools/kernel_probe.py --only apply --m 32000000 --k 64 --reps 1
full trmm_k64 gemm_kernel python tools/kernel_probe.py --only apply --m 32000000 --k 64 --reps 1
full update_q256 update_pass_kernel python tools/kernel_probe.py --only update --m 8000000 --q 256 --k 16 --reps 1
full update_q64 update_pass_kernel python tools/kernel_probe.py --only update --m 8000000 --q 64 --k 16 --reps 1
# the k = 256 factor launch (the second one: after the probe's warm-up call)
"python" tools/kernel_probe.py --only factor --fk 256 --reps 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:factor_kernel --launch-skip 1 -c 1 \
      -o gpurun_out/prof/factor_k256 python tools/kernel_probe.py --only factor --fk 256 --reps 1 > gpurun_out/prof/factor_k256.log 2>&1
ls -la gpurun_out/prof
