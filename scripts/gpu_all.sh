# One gpurun call: build, smoke, GPU parity tests, bench, ncu launch list + one full capture.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
python paper_2406_17565_b200/build.py
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
ls -la gpurun_out
