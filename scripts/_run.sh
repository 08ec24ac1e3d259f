timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python scripts/step_seconds.py config0 10
python bench.py --config config0 --no-cpu-baseline --steps 10
