timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/time_step.py --p 5 --reps 5
