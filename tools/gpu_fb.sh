mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for fb in 64 16 8; do echo "front batches $fb"; SOFA_FRONT_BATCHES=$fb timeout 600 python tools/bimodal_probe.py 2>&1 | head -4; done
