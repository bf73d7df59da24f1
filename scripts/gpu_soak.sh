# gpurun: soak runs of the round-2 protocol -- long two-process bench (pipelined,
# merged copies, host-raised prepares, pruned join queues) and a long ReAct
# full-duplex run with the checksummed pass, plus a 5000-step N=1 bench.
set -x
mkdir -p gpurun_out
TAG=${TAG:-soak}
python paper_2406_17565_b200/build.py
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29677 bench.py --gpus 2 --steps 2000 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
  --pool-blocks 2048 --no-extras > gpurun_out/bench_${TAG}_2p_2000.json 2> gpurun_out/bench_${TAG}_2p_2000.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29678 scripts/workloads_mp.py react --pool-blocks 2048 --sessions 256 --window 8 --check --check-sessions 16 \
  --device 0 --dist-backend gloo > gpurun_out/wmp_${TAG}_react2_256.json 2> gpurun_out/wmp_${TAG}_react2_256.err
timeout 900 python bench.py --steps 5000 --no-extras --no-cpu-baseline > gpurun_out/bench_${TAG}_5000.json 2> gpurun_out/bench_${TAG}_5000.err
