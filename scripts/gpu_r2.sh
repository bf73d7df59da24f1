# Round-2 measurement call: build, smoke, GPU tests, bench and the workload
# drivers with launch overlap on and off (MP_PDL_OVERLAP=0: every migration
# waits for the previous grid, the round-1 behaviour).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'TAG=r2a bash scripts/gpu_r2.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
if [ "${TESTS:-1}" = "1" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
fi
if [ "${BENCH:-1}" = "1" ]; then
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
MP_PDL_OVERLAP=0 timeout 900 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_${TAG}_nooverlap.json 2> gpurun_out/bench_${TAG}_nooverlap.err
for w in loogle react; do
  timeout 300 python scripts/workloads_bench.py $w > gpurun_out/${w}_$TAG.json 2>&1
  MP_PDL_OVERLAP=0 timeout 300 python scripts/workloads_bench.py $w > gpurun_out/${w}_${TAG}_nooverlap.json 2>&1
done
timeout 300 python scripts/sweeps.py chain > gpurun_out/chain_$TAG.json 2>&1
fi
ls -la gpurun_out
