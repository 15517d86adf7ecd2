#!/bin/bash
# Multi-rank host-pipeline hang probe (2 GPUs): the round-1 bench hang (352^3 bs 22, 1x2, beta = 0) under
# several stream-connection settings, plus the mp_worker host cases.  Every command runs under its own
# timeout (process group killed), so a hang costs one line, not the call.
set -u
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
OUT=gpurun_out/hang_probe.txt
: > $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1"
run() {  # name timeout env... -- cmd
  local name=$1 to=$2; shift 2
  local t0=$(date +%s)
  env "$@" > gpurun_out/hp_$name.log 2>&1
  local rc=$?
  echo "$name rc=$rc secs=$(( $(date +%s) - t0 ))" | tee -a $OUT
}
run bench_s352_default 150 timeout -k 5 120 $TR --master-port=29601 bench.py --gpus 2 --config s352 --steps 3 --warmup 3
run bench_s352_conn32 150 CUDA_DEVICE_MAX_CONNECTIONS=32 timeout -k 5 120 $TR --master-port=29602 bench.py --gpus 2 --config s352 --steps 3 --warmup 3
run bench_s352_conn1 150 CUDA_DEVICE_MAX_CONNECTIONS=1 timeout -k 5 120 $TR --master-port=29603 bench.py --gpus 2 --config s352 --steps 3 --warmup 3
run bench_s352_nopipe 150 DBM_HOST_PIPE=0 timeout -k 5 120 $TR --master-port=29604 bench.py --gpus 2 --config s352 --steps 3 --warmup 3
run mp_host 300 DBM_CASE_TIMEOUT=30 timeout -k 5 280 $TR --master-port=29605 tests/mp_worker.py --groups host
run mp_host_conn32 300 CUDA_DEVICE_MAX_CONNECTIONS=32 DBM_CASE_TIMEOUT=30 timeout -k 5 280 $TR --master-port=29606 tests/mp_worker.py --groups host
run mp_sweep 400 DBM_CASE_TIMEOUT=30 timeout -k 5 380 $TR --master-port=29607 tests/mp_worker.py --groups sweep
nvidia-smi --query-gpu=index,name,clocks.sm --format=csv >> $OUT
