# full GPU test suite + smoke (what the driver runs at round end)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -q -m gpu -x --durations=15 2>&1 | tail -40
