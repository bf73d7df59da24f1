# gpurun: does a migration grid smaller than the GPU help back-to-back
# launches (the next grid's CTAs start on the SMs the running one leaves
# free)?  Short-launch chains, the ReAct-like workload and the default bench
# at several CTA caps.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/gpu_r2_ctas.sh'
set -x
mkdir -p gpurun_out
python paper_2406_17565_b200/build.py > /dev/null 2>&1
for c in 0 96 112 128; do
  timeout 300 python scripts/short_launch.py --max-ctas $c --sizes 1,4,8,16,32 --tag cap$c >> gpurun_out/ctas_short.jsonl 2> gpurun_out/ctas_short_$c.err
  timeout 300 python scripts/workloads_bench.py react --max-ctas $c > gpurun_out/ctas_react_$c.json 2> gpurun_out/ctas_react_$c.err
  timeout 300 python bench.py --max-ctas $c --no-extras --no-cpu-baseline > gpurun_out/ctas_bench_$c.json 2> gpurun_out/ctas_bench_$c.err
done
ls -la gpurun_out
