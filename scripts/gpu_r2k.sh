# gpurun: full round-2 check -- build, smoke, every GPU test, the default
# bench line, the two-process line, and the ncu launch list + one full
# capture of the dominant kernel in the bench's configuration.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2k}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29633 bench.py --gpus 2 --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
  --pool-blocks 2048 > gpurun_out/bench_${TAG}_2p_fused.json 2> gpurun_out/bench_${TAG}_2p_fused.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 2 -o gpurun_out/prof_${TAG}_bulk python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_bulk.log 2>&1
ls -la gpurun_out
