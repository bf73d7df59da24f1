# gpurun: batch flush on the host's drain estimate (LaunchTrack::busy_until)
# vs idle-only flush (MP_DRAIN_LEAD_US=0 is not a knob: compare with the
# previous profiles) -- default bench x3, ReAct / LooGLE, coalescing stress tests.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash scripts/gpu_r2_drain.sh'
set -x
mkdir -p gpurun_out
python paper_2406_17565_b200/build.py > /dev/null 2>&1
for r in 1 2 3; do timeout 300 python bench.py --no-extras --no-cpu-baseline > gpurun_out/drain_bench_$r.json 2>/dev/null; done
timeout 300 python scripts/workloads_bench.py react > gpurun_out/drain_react.json 2>/dev/null
timeout 300 python scripts/workloads_bench.py loogle > gpurun_out/drain_loogle.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/pytest_drain.log 2>&1; echo rc=$? >> gpurun_out/pytest_drain.log
