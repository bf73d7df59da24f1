# gpurun: host-time breakdowns of the latency-bound cases (configs[0] tiny
# transfer_with_insert, configs[3] ReAct-like loop).  (compute-sanitizer is
# closed on this GPU pool in round 2: the memcheck of the round-2 kernels is
# profiles/sanitize_memcheck_r02.log, taken before it closed.)
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'TAG=r2s bash scripts/gpu_r2_checks.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2s}
python paper_2406_17565_b200/build.py
MP_HOST_TIMING=1 timeout 300 python scripts/sweeps.py tiny > gpurun_out/tiny_$TAG.json 2> gpurun_out/tiny_$TAG.err
timeout 300 python scripts/sweeps.py tiny > gpurun_out/tiny_${TAG}_notiming.json 2>&1
MP_HOST_TIMING=1 timeout 300 python scripts/workloads_bench.py react --phase-times > gpurun_out/react_phases_$TAG.json 2> gpurun_out/react_phases_$TAG.err
ls -la gpurun_out
