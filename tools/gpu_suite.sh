# full GPU test suite (as the driver runs it) + smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/suite.log 2>&1; echo "gpu suite rc=$?"; tail -3 gpurun_out/suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
