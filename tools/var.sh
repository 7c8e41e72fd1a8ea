python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python tools/kbench.py --variant iterative,hybrid,comparison --n 16777216 --reps 2 2>&1 | grep -v "^{"
python tools/kbench.py --variant hybrid --strict --n 16777216 --reps 2 2>&1 | grep -v "^{"
python tools/kbench.py --variant iterative,hybrid,comparison --dtype f32 --n 16777216 --reps 2 2>&1 | grep -v "^{"
