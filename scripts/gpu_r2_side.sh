# gpurun: the SURVEY §8(f) side measurements and latency sweeps re-run on the
# last round-2 build (round 1 measured them on its own build).
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'TAG=r2x bash scripts/gpu_r2_side.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2x}
python paper_2406_17565_b200/build.py
timeout 600 python scripts/bylayer_study.py > gpurun_out/bylayer_$TAG.json 2> gpurun_out/bylayer_$TAG.err
timeout 600 python scripts/tp_bench.py > gpurun_out/tp_$TAG.json 2> gpurun_out/tp_$TAG.err
for s in swap dram_source gs chain api nccl transfer; do
  timeout 600 python scripts/sweeps.py $s > gpurun_out/sweep_${s}_$TAG.json 2> gpurun_out/sweep_${s}_$TAG.err
done
ls -la gpurun_out
