set -x
python scripts/probe_ab.py /root/repo/abA /root/repo
export GMAF_LAUNCH_MODE=stream
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python scripts/sanitize.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_synccheck.log | head -1) $(grep -c 'sanitize run done' gpurun_out/san_synccheck.log)"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "persistent or c1_parity or ragged or c3_full_size" > gpurun_out/pt30.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt30.log
