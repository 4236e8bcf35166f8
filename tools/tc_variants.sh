#!/bin/bash
# Build timing variants of liblowrank_b200 into build/var_<name>/ from
# NAME=FLAGS pairs, e.g.  tools/tc_variants.sh dbg1="-DLR_TC_DBG=1" sl="-DLR_P_SLEEP=1"
# (run tools/tc_pass_probe.py with LOWRANK_B200_LIB=build/var_<name>/liblowrank_b200.so)
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%=*}"; flags="${spec#*=}"
  python - "$name" $flags <<'PY'
import sys
from paper_0909_4061_b200.build import build
name, flags = sys.argv[1], sys.argv[2:]
build(extra=flags, out=f"build/var_{name}/liblowrank_b200.so", obj=f"build/var_{name}/obj")
PY
done
