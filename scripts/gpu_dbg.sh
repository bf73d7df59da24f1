set -x
mkdir -p gpurun_out
python paper_2406_17565_b200/build.py
timeout 150 python scripts/debug_mp.py golden ce-staged > gpurun_out/dbg3.log 2>&1
MP_REMOTE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29612 scripts/workloads_mp.py react --pool-blocks 2048 --sessions 32 --device 0 --dist-backend gloo --prof \
  > gpurun_out/wmp_r2g_react2.json 2> gpurun_out/wmp_r2g_react2.err
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q --timeout 600 > gpurun_out/pytest_mp_r2g.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mp_r2g.log
