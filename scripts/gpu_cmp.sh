# gpurun: build, GPU parity tests, then bench with each copy engine.
set -x
mkdir -p gpurun_out
TAG=${TAG:-cmp}
python paper_2406_17565_b200/build.py
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --copy-kernel 1 --no-cpu-baseline > gpurun_out/bench_${TAG}_vec.json 2> gpurun_out/bench_${TAG}_vec.err
timeout 900 python bench.py --copy-kernel 2 --no-cpu-baseline --no-swap > gpurun_out/bench_${TAG}_bulk.json 2> gpurun_out/bench_${TAG}_bulk.err
ls -la gpurun_out
