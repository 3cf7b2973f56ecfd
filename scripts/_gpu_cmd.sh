timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --sharded --steps 3 --warmup 3 2>&1 | tail -2
