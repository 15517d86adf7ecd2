cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
OUT=gpurun_out/d4.txt; : > $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1"
run() { local name=$1 to=$2; shift 2; local t0=$(date +%s); timeout -k 10 $to "$@" > gpurun_out/d4_$name.log 2>&1; echo "$name rc=$? secs=$(( $(date +%s) - t0 ))" | tee -a $OUT; }
run nvlink_rate 120 python tools/microbench/nvlink_range.py
run ncu_nvlink 600 /usr/local/cuda/bin/ncu --replay-mode app-range --metrics nvlrx__bytes.sum,nvltx__bytes.sum,gpu__time_duration.sum --csv python tools/microbench/nvlink_range.py
run r64 600 $TR --master-port=29621 bench.py --gpus 4 --config r64 --steps 6 --warmup 3 --no-e2e --timeline gpurun_out/d4_tl_r64
run r64_conn32 600 env CUDA_DEVICE_MAX_CONNECTIONS=32 $TR --master-port=29622 bench.py --gpus 4 --config r64 --steps 6 --warmup 3 --no-e2e --timeline gpurun_out/d4_tl_r64c32
run r64_ts 600 $TR --master-port=29623 bench.py --gpus 4 --config r64 --algorithm tallskinny --steps 6 --warmup 3 --no-e2e --timeline gpurun_out/d4_tl_r64ts
