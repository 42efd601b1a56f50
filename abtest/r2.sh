bash abtest/run.sh; bash abtest/run.sh
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
