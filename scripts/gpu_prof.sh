# one ncu --set full capture of a kernel family (after warmup), report in gpurun_out/
#   bash scripts/gpu_prof.sh <kernel-regex> <skip> <count> [extra bench args]
K=${1:-k_radix}
shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-3} -c ${COUNT:-1} \
  -o gpurun_out/prof_$K python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$K.log 2>&1
tail -2 gpurun_out/ncu_$K.log
