bash abtest/run2.sh; bash abtest/run2.sh
timeout 1400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
