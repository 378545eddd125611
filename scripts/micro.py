import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_25068_b200 as P
lib = P.load(); r = np.zeros(2)
for w, name in [(0, "gumbel"), (5, "rng uniform"), (1, "log"), (2, "exp"), (3, "div"), (4, "L2 chase"), (6, "gumbel_sl"), (7, "5x gumbel_sl"), (8, "log_sl"), (9, "rng_final"), (10, "5x gumbel_sl_v")]:
    lib.dtg_debug_microbench(w, 2000, 1, r); print(f"{name:12s} {r[0]:8.1f} cycles/op")
for g in (2, 16, 66, 148):
    lib.dtg_debug_microbench(100, 2000, g, r); print(f"grid.sync x{g:3d} CTAs {r[0]:8.1f} cycles")
