# gpurun: the round-2 evidence in one call -- build, smoke, every GPU test,
# the default bench line, the process layouts on the one GPU, the workload
# drivers, and ncu (launch list + a full capture of large migration launches).
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'TAG=r2z bash scripts/gpu_r2_final.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2z}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
if [ "${TESTS:-1}" = "1" ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
b() { name=$1; n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline \
    --pool-blocks 2048 "$@" > gpurun_out/bench_${TAG}_$name.json 2> gpurun_out/bench_${TAG}_$name.err; }
b 2p_fused 2
b 4p_fused 4 --no-extras
b 8p_fused 8 --no-extras --pool-blocks 1024
w() { name=$1; n=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + RANDOM % 400)) scripts/workloads_mp.py "$@" --device 0 --dist-backend gloo \
    > gpurun_out/wmp_${TAG}_$name.json 2> gpurun_out/wmp_${TAG}_$name.err; }
w loogle4 4 loogle --pool-blocks 2300 --sessions 2 --check --check-sessions 1
w react8 8 react --pool-blocks 1400 --window 2 --sessions 16 --check --check-sessions 4
w react2 2 react --pool-blocks 2048 --sessions 32 --check
for wl in loogle react; do
  timeout 300 python scripts/workloads_bench.py $wl > gpurun_out/${wl}_$TAG.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate --launch-skip 6 -c 4 -o gpurun_out/prof_${TAG}_bulk python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_full_${TAG}_bulk.log 2>&1
ls -la gpurun_out
