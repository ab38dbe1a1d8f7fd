# A/B timing of ab/libpvr_<name>.so builds against the in-tree library (bench.py c3, no extras)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  if [ $v = base ]; then so=$PWD/paper_1611_07289_b200/libpvr.so; else so=$PWD/ab/libpvr_$v.so; fi
  PVR_SO=$so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ab_$v.log 2>&1
  python -c "
import json,sys;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);k=d['kernels'];print('$v',round(d['ms_per_step'],3),{n:round(k[n]['ms'],3) for n in k})"
done
