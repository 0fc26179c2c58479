#!/bin/bash
# Round-end evidence on one B200 (via gpurun): bench lines of every config, c5 serving, the Table 6 search, and the
# ncu launch list + one full capture of config 4's kernels.  Outputs in gpurun_out/ (scratch); copy the ones to keep
# into profiles/.
cd $GRAFT_REPO_ROOT
OUT=gpurun_out
mkdir -p $OUT
nproc > $OUT/host_nproc.txt; cat /sys/fs/cgroup/cpu.max >> $OUT/host_nproc.txt 2>/dev/null
for cfg in c1 c6; do
  timeout 600 python -u bench.py --config $cfg --steps 50 --warmup 10 --no-serving > $OUT/bench_${cfg}.log 2>&1; echo "bench $cfg rc=$?"
done
timeout 900 python -u bench.py --config c4 --steps 10 --warmup 3 --no-serving > $OUT/bench_c4.log 2>&1; echo "bench c4 rc=$?"
timeout 1500 python -u bench.py --config c3s --sharded --steps 10 --warmup 3 --no-serving > $OUT/bench_c3s.log 2>&1; echo "bench c3s rc=$?"
timeout 300 python -u bench_serving.py --duration 3 > $OUT/serving.log 2>&1; echo "serving rc=$?"
timeout 2400 python -u bench_saturation.py > $OUT/saturation.log 2>&1; echo "saturation rc=$?"
