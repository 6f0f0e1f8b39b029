# ncu evidence (one GPU, never multi-rank).  KREGEX selects the kernel, TAG names the files.
set -x
OUT=gpurun_out
TAG=${TAG:-sr}
KREGEX=${KREGEX:-k_sr}
CFG=${CFG:-C3}
export GMAF_LAUNCH_MODE=stream
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_${TAG}.csv \
  python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline > $OUT/launches_${TAG}.log 2>&1
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 6 -c 1 \
  -o $OUT/prof_${TAG} python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline > $OUT/prof_${TAG}.log 2>&1
ls -la $OUT
