"""Per-kernel counts of the SASS mnemonics that prove tcgen05 / TMEM / TMA /
packed-fp32 use, plus register / shared / local usage, from the built objects.

python tools/sass_evidence.py > profiles/rNN_sass_evidence.txt
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2303_00319_b200", "_lib", "obj")
PAT = re.compile(r"\b(UTC[A-Z]*MMA[A-Z0-9._]*|UTCBAR[A-Z0-9._]*|UTMALDG[A-Z0-9._]*|UTMASTG[A-Z0-9._]*|UTMAPF[A-Z0-9._]*|"
                 r"UBLKCP[A-Z0-9._]*|UBLKPF[A-Z0-9._]*|UTMACCTL[A-Z0-9._]*|"
                 r"LDTM[A-Z0-9._]*|STTM[A-Z0-9._]*|SYNCS\.[A-Z0-9._]*|FMUL2|FFMA2|FADD2|FMNMX3|HMMA[A-Z0-9._]*)\b")
KERNELS = ("k_match_gemm", "k_desc_main", "k_rows_pc_tma", "k_rows_amp0_tma", "k_cols", "k_rows_pc",
           "k_rows_amp0", "k_fast_nms", "k_med_collect")
print("# SASS evidence (cuobjdump -sass of the committed build; mnemonics per the B200 profiling guide)")
for obj in ("match.o", "describe.o", "fields.o", "detect.o"):
    sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", os.path.join(OBJ, obj)], capture_output=True, text=True).stdout
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function ([^ :]+)", line)
        if m:
            cur = m.group(1)
        elif cur and "REG:" in line:
            usage[cur] = " ".join(re.findall(r"(?:REG|SHARED|LOCAL):\d+", line))
    funcs = re.split(r"\n\s*Function : ", sass)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        short = next((k for k in KERNELS if k in name), None)
        if short is None or ("ILi32" not in name and short in ("k_cols", "k_rows_pc", "k_rows_amp0")
                              and "_tma" not in name):
            continue
        if short == "k_rows_pc" and "_tma" not in name and "Li4E" not in name:
            continue
        cnt = collections.Counter(m.group(1).split(".")[0] if not m.group(1).startswith("SYNCS") else m.group(1)
                                  for m in PAT.finditer(f))
        print(f"## {short}  ({name[:70]})  {usage.get(name, '')}")
        for k, v in sorted(cnt.items(), key=lambda kv: -kv[1]):
            print(f"   {v:6d}  {k}")
