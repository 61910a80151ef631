"""Per-kernel SASS instruction-class counts of the built library (cuobjdump -sass):
TMA bulk copies (UBLKCP), bulk prefetch (UBLKPF), mbarrier ops (SYNCS), grid/CTA
barriers, atomics, and the absence of tensor-core MMA (no contraction on this path).

usage: python tools/sass_counts.py [lib.so] > profiles/r2_sass_counts.json
"""
import collections
import json
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2005_12648_b200/libparmerge_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
counts = collections.OrderedDict()
cur = None
pat = {"UBLKCP": r"\bUBLKCP\b", "UBLKPF": r"\bUBLKPF\b", "UTMALDG": r"\bUTMALDG\b", "SYNCS": r"\bSYNCS\.",
       "BAR": r"\bBAR\.", "ATOM/RED": r"\b(ATOMG|ATOM|RED)\.", "LDS": r"\bLDS\b", "STS": r"\bSTS\b",
       "MMA(any)": r"\b(UTC\w*MMA|HMMA|IMMA|QMMA|OMMA)\b"}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur and re.search(r"/\*[0-9a-f]{4,}\*/", line):
        counts[cur]["instructions"] += 1
        for k, p in pat.items():
            if re.search(p, line):
                counts[cur][k] += 1


def short(name):
    r = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return r or name


res = {short(k): dict(v) for k, v in counts.items() if "k_flow" in k or "k_engine" in k or "k_buffered" in k
       or "k_slide" in k or "k_merge" in k or "k_cyc" in k or "k_reverse" in k or "k_gather" in k}
json.dump({"library": lib, "kernels": res}, sys.stdout, indent=1)
