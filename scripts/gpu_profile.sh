# gpurun: bench with each copy engine + ncu launch list + one full ncu capture
# of the dominant kernel (coalesced fused gather->store) in the bench's
# configuration.  Results land in gpurun_out/ (copy summaries to profiles/).
set -x
mkdir -p gpurun_out
TAG=${TAG:-prof}
python paper_2406_17565_b200/build.py
timeout 900 python bench.py --copy-kernel 1 > gpurun_out/bench_${TAG}_vec.json 2> gpurun_out/bench_${TAG}_vec.err
timeout 900 python bench.py --copy-kernel 2 --no-cpu-baseline --no-swap > gpurun_out/bench_${TAG}_bulk.json 2> gpurun_out/bench_${TAG}_bulk.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 2 -o gpurun_out/prof_${TAG}_vector python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --copy-kernel 1 > gpurun_out/ncu_full_${TAG}_vector.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:migrate -c 2 -o gpurun_out/prof_${TAG}_bulk python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline --copy-kernel 2 > gpurun_out/ncu_full_${TAG}_bulk.log 2>&1
ls -la gpurun_out
