set -e
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/r01n_bench.log 2> gpurun_out/r01n_bench.err
tail -1 gpurun_out/r01n_bench.log
echo done
