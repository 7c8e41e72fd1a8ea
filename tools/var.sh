for r in 1 2; do for v in variants/lib_base.so variants/lib_x2.so; do
  TC_LIB_PATH=$v python tools/kbench.py --variant iterative --n 16777216 --reps 3 2>&1 | grep -v "^{" | tail -2 | sed "s|^|$v |"
done; done
