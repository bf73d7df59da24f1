# gpurun: L2 cache-policy hints on the bulk engine (MP_BULK_HINT) -- bench
# line and back-to-back chains, A/B against no hint, twice each.
set -x
mkdir -p gpurun_out
TAG=${TAG:-hint}
python paper_2406_17565_b200/build.py
for rep in 1 2; do
for h in 0 1 2 3; do
  MP_BULK_HINT=$h timeout 300 python bench.py --steps 300 --no-extras --no-cpu-baseline > gpurun_out/bench_${TAG}_h${h}_$rep.json 2>/dev/null
done
done
for h in 0 1 2 3; do
  MP_BULK_HINT=$h timeout 300 python scripts/short_launch.py --tag h$h --sizes 8,32,128 >> gpurun_out/short_$TAG.jsonl 2>/dev/null
done
