"""L2-resident read bandwidth vs buffer size (ct_peak_l2_read): python tools/l2bw.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1402_4381_b200 import ctlib  # noqa: E402
for mib in (4, 8, 16, 24, 32, 48, 64, 96, 1024):
    print(mib, "MiB read %.0f GB/s" % ctlib.ct_peak_l2_read(0, mib, 200 if mib <= 96 else 5))
