# gpurun: last round-2 check on the final code -- GPU suite, smoke, default
# bench (full line), the reference arm, configs[0] latency.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'TAG=r2l bash scripts/gpu_r2_last.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2l}
python paper_2406_17565_b200/build.py > /dev/null 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
timeout 300 python scripts/sweeps.py tiny > gpurun_out/tiny_$TAG.json 2> gpurun_out/tiny_$TAG.err
