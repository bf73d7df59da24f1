set -x
mkdir -p gpurun_out
TAG=${TAG:-r2m}
python paper_2406_17565_b200/build.py
b() { name=$1; n=$2; shift 2
  MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
    --pool-blocks 2048 "$@" > gpurun_out/bench_${TAG}_$name.json 2> gpurun_out/bench_${TAG}_$name.err; }
b 2p_fused 2
b 2p_fused_nopipe 2 --no-extras --no-pipeline
b 4p_fused 4 --no-extras
timeout 1500 python -m pytest tests/test_gpu_multiproc.py -q --timeout 600 > gpurun_out/pytest_mp_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mp_$TAG.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29655 scripts/workloads_mp.py react --pool-blocks 2048 --sessions 32 --check --device 0 --dist-backend gloo \
    > gpurun_out/wmp_${TAG}_react2.json 2> gpurun_out/wmp_${TAG}_react2.err
