TC_LIB_PATH=variants/lib_h1.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fast" 2>&1 | tail -1
for r in 1 2; do for v in variants/*.so; do
  TC_LIB_PATH=$v python tools/kbench.py --variant iterative,hybrid --n 16777216 --reps 3 2>&1 | grep -v "^{" | tail -4 | sed "s|^|$v |"
done; done
