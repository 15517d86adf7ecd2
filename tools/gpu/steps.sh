#!/bin/bash
# One-GPU measurement steps, each under its own timeout, logs in gpurun_out/s_<step>.log and a summary
# line per step in gpurun_out/steps.txt.  Usage (on the GPU box, via gpurun):
#   bash tools/gpu/steps.sh tests bench:sq64 bench:sq22:blocked ncu_smm22q dgemm_sweep ...
# Steps:
#   tests                 pytest -m gpu (the driver's GPU tier) + smoke()
#   bench:<cfg>[:<path>]  bench.py --config cfg [--path path] --steps 3 --warmup 3 (JSON line -> s_bench_*.json)
#   ncu_smm22q            ncu --set full of the bs-22 square kernel at 5,632^3 (one launch)
#   ncu_dgemm_traffic     ncu dram bytes of one bench-shape dgemm launch (63,360 x 63,360 x 16,896: a K-chunk)
#   ncu_dgemm_full        ncu --set full of one bench-shape dgemm launch
#   dgemm_sweep           bench-shape dgemm time under DBM_DGEMM_WAVESYNC / _WAVESLACK settings
#   launches:<cfg>[:path] ncu launch list (gpu__time_duration) of one bench step
set -u
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
SUM=gpurun_out/steps.txt
NCU=/usr/local/cuda/bin/ncu
step() {  # name seconds cmd...
  local name=$1 to=$2; shift 2
  local t0=$(date +%s)
  timeout -k 10 $to "$@" > gpurun_out/s_$name.log 2>&1
  local rc=$?
  echo "$name rc=$rc secs=$(( $(date +%s) - t0 ))" | tee -a $SUM
  return $rc
}
for s in "$@"; do
  IFS=: read -r kind a b c <<< "$s"
  case $kind in
    tests)
      step pytest 1500 python -m pytest tests -m gpu -x -q
      step smoke 300 python -c "import __graft_entry__ as g; g.smoke()" ;;
    bench)
      nm=bench_${a}${b:+_$b}${c:+_$c}
      if [ -n "$c" ]; then envs="$c"; else envs=""; fi
      step $nm 1500 env $envs python bench.py --config $a ${b:+--path $b} --steps 3 --warmup 3
      tail -1 gpurun_out/s_$nm.log > gpurun_out/s_$nm.json ;;
    ncu_smm22q)
      step ncu_smm22q 900 $NCU --set full --import-source on --clock-control none -k regex:smm22q -c 1 \
        -o gpurun_out/ncu_smm22q -f python tools/profile_multiply.py --M 5632 --N 5632 --K 5632 --bs 22 --reps 1 ;;
    ncu_dgemm_traffic)
      for ws in ${WAVES:-0}; do
        step ncu_dgemm_ws$ws 1200 env DBM_DGEMM_WAVESYNC=$ws $NCU --clock-control none -k regex:dgemm_tn -c 1 \
          --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
          --csv python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 1
      done ;;
    ncu_nu_smm)
      step ncu_nu_smm 900 $NCU --set full --import-source on --clock-control none -k regex:nu_smm -c 1 \
        -o gpurun_out/ncu_nu_smm -f python bench.py --config nus --path blocked --steps 1 --warmup 0 --no-e2e \
        --no-cpu-baseline ;;
    ncu_dgemm_full)
      step ncu_dgemm_full 1500 $NCU --set full --import-source on --clock-control none -k regex:dgemm_tn -c 1 \
        -o gpurun_out/ncu_dgemm_full -f python tools/profile_dgemm.py --M 63360 --N 63360 --K 16896 --reps 1 ;;
    dgemm_sweep)
      SW="${SWEEP:-0:1 32:1 64:1 128:1 64:2 16:1}"
      for cfg in $SW; do
        IFS=: read -r ws sl <<< "$cfg"
        step dgemm_ws${ws}_sl${sl} 600 env DBM_DGEMM_WAVESYNC=$ws DBM_DGEMM_WAVESLACK=$sl \
          python tools/profile_dgemm.py --M 63360 --N 63360 --K 15872 --reps 4
      done ;;
    launches)
      nm=launches_${a}${b:+_$b}
      step $nm 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/$nm.csv python bench.py --config $a ${b:+--path $b} --steps 1 --warmup 1 \
        --no-e2e --no-cpu-baseline ;;
    *) echo "unknown step $s" | tee -a $SUM ;;
  esac
done
nvidia-smi --query-gpu=index,name,clocks.sm,clocks_event_reasons.active --format=csv >> $SUM
