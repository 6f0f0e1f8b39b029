# ncu evidence for the PCG kernels at C3 (one GPU, never multi-rank).
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
# launch list with device times: one C3 step (cold-cache, serialised: compare shares)
GMAF_LAUNCH_MODE=stream timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/launches_bench.log 2>&1
# full set on the two iteration kernels (a few launches after warm-up)
GMAF_LAUNCH_MODE=stream timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_phase_b -s 40 -c 1 \
  -o $OUT/prof_phase_b python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/prof_b.log 2>&1
GMAF_LAUNCH_MODE=stream timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_phase_a -s 40 -c 1 \
  -o $OUT/prof_phase_a python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/prof_a.log 2>&1
ls -la $OUT
