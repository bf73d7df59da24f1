# gpurun: the multi-process GPU tests only (no -x: every failure reported)
set -x
mkdir -p gpurun_out
TAG=${TAG:-mpt}
python paper_2406_17565_b200/build.py
timeout 1500 python -m pytest tests/test_gpu_multiproc.py -q --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_mp_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mp_$TAG.log
