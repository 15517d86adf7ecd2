#!/bin/bash
# Multi-rank validation on the GPUs of one box (2 or 4): the host-pipeline cases first (they hung in
# round 1), then the whole mp_worker parity suite with its JSON summary, then bench lines.  Each command
# runs under its own timeout; results land in gpurun_out/mg_<n>gpu_*.
set -u
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/mg_${N}gpu.txt
: > $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1"
run() {  # name seconds cmd...
  local name=$1 to=$2; shift 2
  local t0=$(date +%s)
  timeout -k 10 $to "$@" > gpurun_out/mg_${N}gpu_$name.log 2>&1
  local rc=$?
  echo "$name rc=$rc secs=$(( $(date +%s) - t0 ))" | tee -a $OUT
}
run nvlink_rate 120 python tools/microbench/nvlink_range.py
run ncu_nvlink 600 /usr/local/cuda/bin/ncu --replay-mode app-range \
    --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum --csv python tools/microbench/nvlink_range.py
run bench_s352 150 $TR --master-port=29611 bench.py --gpus $N --config s352 --steps 3 --warmup 3
run mp_host 600 env DBM_CASE_TIMEOUT=60 $TR --master-port=29612 tests/mp_worker.py --groups host,sweep \
    --summary gpurun_out/mg_${N}gpu_host_summary.json
run mp_all 1500 env DBM_CASE_TIMEOUT=120 $TR --master-port=29613 tests/mp_worker.py --groups cannon,sparse,host,nonuni \
    --summary gpurun_out/mg_${N}gpu_all_summary.json
# BENCH_SPECS: "cfg" or "name=bench args" (spaces in args as commas), e.g. "sq64 sq64nccl=--config,sq64,--transport,nccl"
for spec in ${BENCH_SPECS:-${BENCH_CFGS:-sq64}}; do
  name=${spec%%=*}
  if [ "$name" = "$spec" ]; then args="--config $spec"; else args=$(echo "${spec#*=}" | tr ',' ' '); fi
  run bench_$name 900 $TR --master-port=29614 bench.py --gpus $N $args --steps 3 --warmup 3 \
      --timeline gpurun_out/mg_${N}gpu_timeline_$name
done
