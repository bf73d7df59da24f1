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
# configs[2] / configs[3] multi-process drivers on the one GPU (content-checked pass)
wmp() {  # $1 = nproc, $2 = name, rest = args
  n=$1; name=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) scripts/workloads_mp.py "$@" --device 0 --dist-backend gloo \
    > gpurun_out/wmp_${TAG}_${name}.json 2> gpurun_out/wmp_${TAG}_${name}.err
  echo "wmp $name rc=$?" >> gpurun_out/mpbench_${TAG}.log
}
if [ "${WMP:-1}" = "1" ]; then
wmp 4 loogle4 loogle --pool-blocks 2300 --sessions 2 --check --check-sessions 1
wmp 8 react8 react --pool-blocks 1400 --window 2 --sessions 16 --check --check-sessions 4
wmp 2 react2 react --pool-blocks 2048 --sessions 32 --check
fi
if [ "${WB:-1}" = "1" ]; then
for w in loogle react; do
  timeout 300 python scripts/workloads_bench.py $w > gpurun_out/${w}_$TAG.json 2>&1
done
fi
ls -la gpurun_out
