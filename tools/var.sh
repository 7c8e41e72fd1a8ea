python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for r in 1 2; do python tools/kbench.py --variant iterative,hybrid --n 16777216 --reps 3 2>&1 | grep -v "^{" | tail -4; done
