set -e
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/r01m_bench_full.log 2> gpurun_out/r01m_bench_full.err
tail -1 gpurun_out/r01m_bench_full.log > gpurun_out/r01m_bench_full.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r01m_bench_reference.log 2>&1
tail -1 gpurun_out/r01m_bench_reference.log > gpurun_out/r01m_bench_reference.json
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-hybrid > gpurun_out/r01m_small.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ --csv --log-file gpurun_out/r01m_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-hybrid > gpurun_out/r01m_ncu_launch.log 2>&1
echo done
