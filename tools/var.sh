for r in 1 2; do for v in variants/*.so; do
  TC_LIB_PATH=$v python tools/kbench.py --variant iterative,hybrid --n 16777216 --reps 3 2>&1 | grep -v "^{" | tail -4 | sed "s|^|$v |"
done; done
