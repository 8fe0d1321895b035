mkdir -p gpurun_out
compute-sanitizer --tool synccheck tools/probes/mbar_synccheck > gpurun_out/probe_synccheck.log 2>&1; echo "probe rc=$?"; tail -5 gpurun_out/probe_synccheck.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest.log
