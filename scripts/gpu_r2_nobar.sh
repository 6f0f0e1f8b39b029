# timing-only experiment: the row pipeline without its two CTA barriers per row (results wrong)
set -x
timeout 600 python scripts/probe_slab_sizes.py > gpurun_out/slab_bar.log 2>&1
GMAF_NVCC_EXTRA=-DGMAF_EXPERIMENT_NOBAR python -c "from paper_2511_06824_b200 import build as B; B.build(force=True)"
timeout 600 python scripts/probe_slab_sizes.py > gpurun_out/slab_nobar.log 2>&1
python -c "from paper_2511_06824_b200 import build as B; B.build(force=True)"
cat gpurun_out/slab_bar.log gpurun_out/slab_nobar.log
