#!/bin/bash
# Build experiment variants of the library: tools/build_variants.sh name:DEF1,DEF2 name2:DEF3 ...
cd "$(dirname "$0")/.."
pids=()
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  python - "$name" "$defs" <<'PY' &
import sys
from paper_2105_12415_b200 import _build
name, defs = sys.argv[1], sys.argv[2]
d = [x for x in defs.split(",") if x and x != name]
_build.build(out=f"variants/{name}.so", defines=d)
print("built", name, d)
PY
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
