"""SASS opcode histogram of the shipped libcvr.so (cuobjdump -sass): proves which kernels run on tcgen05 (UTCHMMA /
UTCBAR / LDTM), TMA (UTMALDG / UTMASTG) and which on legacy mma.sync (HMMA).  Writes profiles/sass_<tag>.json.
usage: python scripts/sass_histogram.py <tag>"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
lib = os.path.join(ROOT, "paper_2605_29232_b200", "libcvr.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "HMMA", "LDSM", "SYNCS", "FFMA", "LDG", "STG"]
total = collections.Counter()
per = {}
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    c = collections.Counter()
    two_cta = 0
    for line in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m:
            c[m.group(1)] += 1
            if m.group(1) == "UTCHMMA" and "2CTA" in line:
                two_cta += 1
    total.update(c)
    short = re.sub(r"^_Z\w*?(gemm_bf16_kernel|embed_bag_kernel|dense_f32_kernel|mha64_v2_kernel|unpack_kernel|"
                   r"head_finalize_kernel|set_call_kernel|peer_\w+_kernel)", r"\1", name)[:120]
    per[short] = {k: c[k] for k in KEYS if c[k]}
    if two_cta:
        per[short]["UTCHMMA_2CTA"] = two_cta
out = {"lib": "paper_2605_29232_b200/libcvr.so", "arch": "sm_100a", "totals": {k: total[k] for k in KEYS},
       "per_kernel": per,
       "note": "UTCHMMA = tcgen05.mma (UTCHMMA...2CTA = cta_group::2), LDTM = tcgen05.ld, UTMALDG/UTMASTG = TMA "
               "tensor loads/stores, HMMA = legacy mma.sync (the c4 attention core, cvr_attn.cuh)"}
p = os.path.join(ROOT, "profiles", f"sass_{tag}.json")
json.dump(out, open(p, "w"), indent=1)
print(json.dumps(out["totals"]))
