# multi-GPU shard path: GPU test suite + the single-GPU cost of the shard code path (world = 1,
# identity all-reduce) against the plain solve on C5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/shard_cost.py c5 5
