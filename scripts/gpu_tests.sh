set -x
UPIPE_PARITY_REPORT=gpurun_out/parity_r02.json timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest exit $?"; tail -12 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
