# gpurun: build, all GPU tests, bench at N=1, and the multi-process (1P1D,
# two processes) bench path on the single GPU of the box.
set -x
mkdir -p gpurun_out
TAG=${TAG:-mp}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/bench_${TAG}_2proc.json 2> gpurun_out/bench_${TAG}_2proc.err
ls -la gpurun_out
