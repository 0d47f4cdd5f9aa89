"""Replay passes of candidate single-pass metric groups (CUPTI host config)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2102_05297_b200 import counters as cc, live
from paper_2102_05297_b200.tuner import Tuner
t = Tuner(0)
g1 = list(live.GROUP1_ABBRS)
cands = {"group1": g1, "group1+SHR_U": g1 + ["SHR_U"],
         "group1-TEX_RWT+SHR_U": [a for a in g1 if a != "TEX_RWT"] + ["SHR_U"],
         "group1-SM_E+SHR_U": [a for a in g1 if a != "SM_E"] + ["SHR_U"],
         "group1-INST_ISSUE_U+SHR_U": [a for a in g1 if a != "INST_ISSUE_U"] + ["SHR_U"],
         "group1-DRAM_U+SHR_U": [a for a in g1 if a != "DRAM_U"] + ["SHR_U"],
         "SHR_U": ["SHR_U"], "all": list(live.TABLE1_ABBRS)}
for k, ab in cands.items():
    ms = [cc.VOLTA_METRICS[a][0] for a in ab]
    print(k, len(ms), "passes", t.profile_passes(ms), flush=True)
for a in live.TABLE1_ABBRS:
    print(" +", a, t.profile_passes([cc.VOLTA_METRICS[x][0] for x in g1 + [a]] if a not in g1 else [cc.VOLTA_METRICS[x][0] for x in g1]), flush=True)
