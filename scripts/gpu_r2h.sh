set -x
mkdir -p gpurun_out
TAG=${TAG:-r2h}
python paper_2406_17565_b200/build.py
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q --timeout 600 > gpurun_out/pytest_mp_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mp_$TAG.log
MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29611 bench.py --gpus 2 --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
  --pool-blocks 2048 --no-extras > gpurun_out/bench_${TAG}_2p_fused.json 2> gpurun_out/bench_${TAG}_2p_fused.err
MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29612 scripts/workloads_mp.py react --pool-blocks 2048 --sessions 32 --device 0 --dist-backend gloo \
  > gpurun_out/wmp_${TAG}_react2.json 2> gpurun_out/wmp_${TAG}_react2.err
