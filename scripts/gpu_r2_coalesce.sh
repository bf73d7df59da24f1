# gpurun: the coalescing limit (payload of one merged migration launch) on
# the default bench, three runs per setting.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash scripts/gpu_r2_coalesce.sh'
set -x
mkdir -p gpurun_out
python paper_2406_17565_b200/build.py > /dev/null 2>&1
for r in 1 2 3; do
  for c in 256 512 1024 2048 4096; do
    timeout 300 python bench.py --coalesce-mib $c --no-extras --no-cpu-baseline > gpurun_out/coal_${c}_$r.json 2> gpurun_out/coal_${c}_$r.err
  done
done
