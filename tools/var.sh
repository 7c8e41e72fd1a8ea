# Time every variants/*.so (TC_LIB_PATH override) with kbench: tools/var.sh [variant-list] [n]
VL=${1:-hybrid}
N=${2:-16777216}
for r in 1 2; do for v in variants/*.so; do
  TC_LIB_PATH=$v python tools/kbench.py --variant $VL --n $N --reps 3 2>&1 | grep -v "^{" | awk 'NR%3==0' | sed "s|^|$v |"
done; done
