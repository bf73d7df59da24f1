# gpurun: the process layouts on one GPU under MPS (the processes' kernels run
# concurrently instead of time-slicing the GPU between contexts), so the
# cross-process protocols that need the receiver's GPU per handoff (STAGED
# unpacks, ReAct's D->P returns) are not charged a context switch each time.
set -x
mkdir -p gpurun_out
TAG=${TAG:-mps}
python paper_2406_17565_b200/build.py
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d; sleep 2
b() { name=$1; n=$2; shift 2
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
    --pool-blocks 2048 --no-extras "$@" > gpurun_out/bench_${TAG}_$name.json 2> gpurun_out/bench_${TAG}_$name.err; }
b 2p_fused 2
b 2p_staged 2 --xfer-path staged
b 4p_fused 4
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29688 scripts/workloads_mp.py react --pool-blocks 2048 --sessions 32 --check --device 0 --dist-backend gloo \
  > gpurun_out/wmp_${TAG}_react2.json 2> gpurun_out/wmp_${TAG}_react2.err
echo quit | nvidia-cuda-mps-control
cat $CUDA_MPS_LOG_DIRECTORY/control.log > gpurun_out/mps_control_$TAG.log 2>&1
