#!/usr/bin/env bash
# Build tuning variants of the library (development): each VAR="name:flags"
# goes to build/var_<name>/liblowrank_b200.so; select one with
# LOWRANK_B200_LIB=... when running a probe.
set -e
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  python - "$name" "$flags" <<'PY'
import sys, os
sys.path.insert(0, "/root/repo")
from paper_0909_4061_b200 import build as b
name, flags = sys.argv[1], sys.argv[2].split()
out = f"/root/repo/build/var_{name}/liblowrank_b200.so"
os.makedirs(os.path.dirname(out), exist_ok=True)
b.build(extra=flags, out=out, obj=f"/root/repo/build/var_{name}/obj")
print(out)
PY
done
