# gpurun: the multi-process bench line (N=2 and N=4 processes on the one GPU
# of the box, gloo bootstrap) for every transport, plus the N=1 default line.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'TAG=r2c bash scripts/gpu_mpbench.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-mpb}
python paper_2406_17565_b200/build.py
run() {  # $1 = nproc, $2 = name, rest = bench args
  n=$1; name=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps ${STEPS:-30} --warmup 3 --device 0 \
    --dist-backend gloo --no-cpu-baseline --pool-blocks 2048 "$@" \
    > gpurun_out/bench_${TAG}_${name}.json 2> gpurun_out/bench_${TAG}_${name}.err
  echo "$name rc=$?" >> gpurun_out/mpbench_${TAG}.log
}
run 2 2p_fused --xfer-path fused
run 2 2p_fused_peer_vector --xfer-path fused --peer-engine 1 --no-extras
run 2 2p_staged --xfer-path staged --no-extras
run 2 2p_ce --xfer-path ce --no-extras
run 4 4p_fused --xfer-path fused --no-extras
if [ "${N1:-1}" = "1" ]; then
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
fi
ls -la gpurun_out
