#!/bin/bash
# Re-capture every ncu artefact summarised under profiles/ (run on the GPU
# box through gpurun; each command first runs without ncu and must exit 0).
#   launch list of the bench command (cold-cache, serialised: compare shares)
#   --set full of K1 (both passes + policy) and K2 at config 1 and K1 at config 4,
#   K3 mid-session at config 1, the diagnostics kernel.
# Then locally: python tools/ncu_summary.py r2 gpurun_out/launches.csv gpurun_out/*.ncu-rep
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --clock-control none"
FULL="$NCU --set full --import-source on"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/pre_bench.json || exit 1
$NCU --metrics gpu__time_duration.sum -c 12000 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > $OUT/ncu_launch.log 2>&1
python tools/profile_targets.py k3 > $OUT/pre_k3.log || exit 1
$FULL -k regex:'k1tc_|k1_policy' -c 3 -o $OUT/k1k2_full -f python tools/profile_targets.py k3 > $OUT/ncu_k1.log 2>&1
$FULL -k regex:'k2_compact' -c 1 -o $OUT/k2_full -f python tools/profile_targets.py k3 > $OUT/ncu_k2.log 2>&1
$FULL -k regex:'k3_decode' -s 200 -c 1 -o $OUT/k3_full -f python tools/profile_targets.py k3 > $OUT/ncu_k3.log 2>&1
python tools/profile_targets.py k3f > $OUT/pre_k3f.log || exit 1
$FULL -k regex:'k3_decode' -s 200 -c 1 -o $OUT/k3f_full -f python tools/profile_targets.py k3f > $OUT/ncu_k3f.log 2>&1
python tools/profile_targets.py diag > $OUT/pre_diag.log || exit 1
$FULL -k regex:'decode_recovery' -s 200 -c 1 -o $OUT/diag_full -f python tools/profile_targets.py diag > $OUT/ncu_diag.log 2>&1
python tools/k1_timing.py c4 > $OUT/pre_c4.log || exit 1
$FULL -k regex:'k1tc_' -c 2 -o $OUT/k1_c4_full -f python tools/k1_timing.py c4 > $OUT/ncu_c4.log 2>&1
ls -la $OUT/*.ncu-rep
