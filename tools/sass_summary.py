"""Per-kernel counts of the instructions that prove the tensor-core / TMA /
TMEM paths in the built library (cuobjdump -sass), for profiles/.

    python tools/sass_summary.py [lib.so] > profiles/roundN_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_0909_4061_b200/liblowrank_b200.so"
KEYS = ["UTCHMMA", "UTCIMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "UTCATOMSWS",
        "DMMA", "HMMA", "SYNCS", "FENCE.VIEW.ASYNC.S"]

out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True,
                     text=True).stdout
cur = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for k in KEYS:
        if re.search(r"\b" + re.escape(k), line):
            counts[cur][k] += 1


def demangle(names):
    p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return p.stdout.splitlines()


names = [n for n, c in counts.items() if sum(c.values())]
pretty = demangle(names)
print(f"# SASS instruction counts per kernel ({LIB}, cuobjdump -sass, sm_100a)")
print("# " + "  ".join(KEYS))
for n, p in zip(names, pretty):
    c = counts[n]
    p = p.replace("(anonymous namespace)::", "").replace("lr::", "").replace("void ", "")
    p = re.sub(r"\(.*", "", p)
    row = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
    print(f"{p[:90]:90s} {row}")
