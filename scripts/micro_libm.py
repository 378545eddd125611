"""Latency (clock64 cycles per dependent op) of the device libm: glibc
restatement vs libdevice, one lane and 32 divergent lanes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2603_25068_b200 as P

names = {0: "gumbel (glibc, 1 lane)", 1: "log libdevice", 2: "exp libdevice", 8: "log_sl (glibc)",
         11: "glibc log table path", 12: "glibc log near-1 path", 13: "glibc exp",
         15: "32 lanes glibc log", 16: "32 lanes libdevice log", 17: "32 lanes gumbel",
         18: "32 lanes 5 interleaved gumbels", 10: "5 interleaved gumbels (1 lane)", 6: "gumbel_sl chain"}
lib = P.load()
for w, nm in names.items():
    r = np.zeros(2)
    assert lib.dtg_debug_microbench(w, 2000, 0, r) == 0
    print(f"{w:3d} {nm:34s} {r[0]:8.1f} cycles")
