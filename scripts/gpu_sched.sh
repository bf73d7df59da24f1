# gpurun: bulk-engine work distribution, static vs dynamic (MP_BULK_SCHED),
# kernel sweep + bench + workloads; GPU parity tests with the default.
mkdir -p gpurun_out
TAG=${TAG:-sched}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
for m in static dynamic; do
  for c in 0 4 5; do MP_BULK_SCHED=$m MP_BULK_CFG=$c timeout 300 python scripts/kernel_sweep.py 2 | sed "s/^/$m cfg$c /"; done
  MP_BULK_SCHED=$m timeout 600 python bench.py --no-extras --no-cpu-baseline > gpurun_out/bench_${TAG}_$m.json 2> gpurun_out/bench_${TAG}_$m.err
  MP_BULK_SCHED=$m timeout 300 python scripts/workloads_bench.py loogle > gpurun_out/wl_loogle_${TAG}_$m.json 2>&1
done > gpurun_out/sweep_$TAG.txt 2>&1
