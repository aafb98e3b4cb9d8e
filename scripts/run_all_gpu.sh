mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/t_all.log 2>&1; echo "pytest rc $?" >> gpurun_out/t_all.log
tail -3 gpurun_out/t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
