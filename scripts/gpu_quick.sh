# quick GPU check: selected tests (PYTEST_K), smoke
set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "${PYTEST_K}" > gpurun_out/gpuquick.log 2>&1; echo "pytest exit $?"; tail -25 gpurun_out/gpuquick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
