# One gpurun call: build, smoke, GPU parity tests, bench, the workload and
# latency side measurements, the multi-process layouts on the one GPU, and the
# ncu launch list + one full capture of the migration kernel.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'TAG=r2a bash scripts/gpu_all.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
if [ "${EXTRA:-1}" = "1" ]; then
for w in loogle react; do timeout 300 python scripts/workloads_bench.py $w > gpurun_out/${w}_$TAG.json 2>&1; done
timeout 300 python scripts/sweeps.py chain > gpurun_out/chain_$TAG.json 2>&1
timeout 300 python scripts/sweeps.py api > gpurun_out/api_$TAG.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/bench_${TAG}_2proc.json 2> gpurun_out/bench_${TAG}_2proc.err
fi
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
ls -la gpurun_out
