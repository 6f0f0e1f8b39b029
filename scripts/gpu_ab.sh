# A/B of kernel variants: env assignments passed as arguments, e.g. bash scripts/gpu_ab.sh "GMAF_SR_COLS=1" "GMAF_SR_COLS=2"
for v in "$@"; do
  env $v timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(round(d['value']/1e9,2),'G', round(d['roofline']['avg_launch_us_events'],1),'us')" 2>&1 | tail -1)"
done
