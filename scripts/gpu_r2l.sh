set -x
mkdir -p gpurun_out
TAG=${TAG:-r2l}
python paper_2406_17565_b200/build.py
b() { name=$1; n=$2; shift 2
  MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
    --pool-blocks 2048 "$@" > gpurun_out/bench_${TAG}_$name.json 2> gpurun_out/bench_${TAG}_$name.err; }
b 2p_fused 2
b 4p_fused 4 --no-extras
b 2p_staged 2 --no-extras --xfer-path staged
b 2p_ce 2 --no-extras --xfer-path ce
b 2p_peer_vector 2 --no-extras --peer-engine 1
