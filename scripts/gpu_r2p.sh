set -x
mkdir -p gpurun_out
TAG=${TAG:-r2p}
python paper_2406_17565_b200/build.py
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_alloc_claims.py -q --timeout 600 -k "pipeline or compaction or claims" > gpurun_out/pytest_new_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new_$TAG.log
timeout 1200 compute-sanitizer --tool memcheck --leak-check no python tests/sanitize_tour.py > gpurun_out/sanitize_memcheck_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck_$TAG.log
MP_HOST_TIMING=1 timeout 300 python bench.py --steps 100 --no-extras --no-cpu-baseline > gpurun_out/bench_hosttiming_$TAG.json 2> gpurun_out/bench_hosttiming_$TAG.err
