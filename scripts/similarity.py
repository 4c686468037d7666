"""Development: token-sequence similarity (difflib ratio, comments and string
literals stripped) of host sources against their reference counterparts."""
import difflib
import re
import sys

PAIRS = [("paper_0710_0510_b200/csrc/host/" + f, "/root/reference/proj/src/" + f)
         for f in ("redq.cpp", "gfq.cpp", "params.cpp", "dqt.cpp", "fpdiv.cpp", "common.cpp", "polymul.cpp")]
PAIRS.append(("tools/qpack_b200.cpp", "/root/reference/proj/tools/qpack.cpp"))


def tokens(path):
    s = open(path).read()
    s = re.sub(r"//[^\n]*", " ", s)
    s = re.sub(r"/\*.*?\*/", " ", s, flags=re.S)
    s = re.sub(r'"(\\.|[^"\\])*"', '"S"', s)
    return re.findall(r"[A-Za-z_]\w*|\d+|\S", s)


for ours, ref in PAIRS:
    try:
        a, b = tokens(ours), tokens(ref)
    except FileNotFoundError as e:
        print(e)
        continue
    sm = difflib.SequenceMatcher(None, a, b, autojunk=False)
    la = set(l.strip() for l in open(ours) if len(l.strip()) > 8)
    lb = set(l.strip() for l in open(ref) if len(l.strip()) > 8)
    print(f"{ours:55s} ratio {sm.ratio():.2f}  identical lines {len(la & lb)}")
