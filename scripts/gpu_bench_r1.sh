set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
python paper_2406_17565_b200/build.py
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 3 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --pool-blocks 2048 > gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out
