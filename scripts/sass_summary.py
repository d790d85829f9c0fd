"""Per-kernel SASS mnemonic counts of the built libarc.so (cuobjdump -sass): the evidence that the hot
kernels are tcgen05 / TMA code (UTCxMMA, UTCCP, LDTM, UTMALDG, UTMASTG, UBLKCP) and that no legacy
HMMA path exists.  Writes profiles/<out>.json."""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2601_07475_b200", "libarc.so")
KEYS = ["UTCQMMA", "UTCHMMA", "UTCOMMA", "UTCMMA", "UTCCP", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP",
        "UTMAPF", "SYNCS", "HMMA", "HGMMA", "QGMMA", "LDGSTS", "ELECT", "REDG", "ATOMG"]


def main(out):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m:
            op = m.group(1)
            full = op + (m.group(2) or "")
            for k in KEYS:
                if op.startswith(k):
                    per[cur][full if k in ("UTCQMMA", "UTCHMMA", "UTCOMMA", "UTCMMA", "UTMALDG") else k] += 1
    res = {}
    for fn, c in per.items():
        demangled = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
        short = re.sub(r"\(.*", "", demangled.replace("(anonymous namespace)::", ""))
        res[short] = dict(sorted(c.items()))
    total = collections.Counter()
    for c in res.values():
        total.update(c)
    doc = {"source": "cuobjdump -sass paper_2601_07475_b200/libarc.so (sm_100a)", "kernels": res,
           "total": dict(sorted(total.items())), "hmma_free": total.get("HMMA", 0) == 0}
    with open(os.path.join(ROOT, "profiles", out), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc["total"]))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2_sass_summary.json")
