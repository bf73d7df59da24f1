mkdir -p gpurun_out
python paper_2406_17565_b200/build.py > /dev/null 2>&1
for c in 4096; do for r in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) bench.py --gpus 2 --steps 30 --warmup 3 --device 0 --dist-backend gloo --no-cpu-baseline --no-extras --pool-blocks 2048 --coalesce-mib $c > gpurun_out/mp2_${c}_$r.json 2> gpurun_out/mp2_${c}_$r.err
done; done
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 600 > gpurun_out/pytest_mp_idle.log 2>&1; echo rc=$? >> gpurun_out/pytest_mp_idle.log
