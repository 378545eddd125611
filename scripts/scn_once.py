"""One scenario-resident (mode 4) C3 forward after a warm-up, for ncu: scn_once.py B [T]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_25068_b200 import _lib
if os.environ.get("DTG_LIB"):  # another build (scripts/build_variants.sh)
    _lib.load_other(os.environ["DTG_LIB"])
import paper_2603_25068_b200 as P
B = int(sys.argv[1]); T = int(sys.argv[2]) if len(sys.argv) > 2 else 120
sc = P.Scenario.grid(23, 1609.34, 42, 1000.0).configure(1000020, 30, T, 300)
p = sc.sample_parameters(3); lk, ps = sc.seed_agents()
e = P.Engine(sc, B, T); e.set_params(p); e.set_state(lk, ps); e.set_mode(4)
for b in range(B): e.set_noise(7, b, b)
e.forward(T, sc.steps_per_interval); e.sync()
e.forward(T, sc.steps_per_interval); e.sync()
print("ok", e.last_mode)
