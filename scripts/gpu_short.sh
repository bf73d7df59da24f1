# gpurun: short-launch sweep of the migration kernel's ring geometry and CTA
# cap (scripts/short_launch.py), one process per setting.
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'TAG=r2d bash scripts/gpu_short.sh'
set -x
mkdir -p gpurun_out
TAG=${TAG:-short}
python paper_2406_17565_b200/build.py
out=gpurun_out/short_$TAG.jsonl
: > $out
s() { timeout 300 env "$@" >> $out 2>> gpurun_out/short_$TAG.err; }
s python scripts/short_launch.py --tag auto
s MP_PDL_OVERLAP=0 python scripts/short_launch.py --tag auto_nooverlap
s MP_BULK_CFG=0 python scripts/short_launch.py --tag 64kx3
s MP_BULK_CFG=1 python scripts/short_launch.py --tag 32kx3
s MP_BULK_CFG=1 python scripts/short_launch.py --tag 32kx3_1persm --max-ctas 148
s MP_BULK_CFG=3 python scripts/short_launch.py --tag 16kx4
s MP_BULK_CFG=3 python scripts/short_launch.py --tag 16kx4_2persm --max-ctas 296
s MP_BULK_CFG=2 python scripts/short_launch.py --tag 8kx6_2persm --max-ctas 296
s MP_BULK_CFG=5 python scripts/short_launch.py --tag 48kx4
ls -la gpurun_out
