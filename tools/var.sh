for r in 1 2; do for v in variants/*.so; do
  TC_LIB_PATH=$v python tools/kbench.py --variant comparison,hybrid --n 16777216 --reps 3 2>&1 | grep -v "^{" | awk 'NR==3||NR==6' | sed "s|^|$v |"
done; done
