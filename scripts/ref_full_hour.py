"""One full 1-hour C3 nowcast (120 steps) of the reference build on this
host's CPU, to validate bench.py's 1-step extrapolation of the reference arm
(VERDICT r1 item 3).  Prints one JSON line."""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from oracle.oracle import RefLib, RefScenario, fnv1a64_c

R = RefLib()
mk = lambda T: RefScenario.grid(R, bench.GRID_N, bench.LINK_LEN, bench.NET_SEED, bench.VIRT_LEN).configure(
    bench.VEHICLES, bench.DELTA_N, T, bench.OBS_S)
s0 = mk(0)
p = s0.sample_parameters(bench.PARAM_SEED)
t = time.perf_counter(); s0.forward(p, bench.SIM_SEED, 0); setup = time.perf_counter() - t
s1 = mk(1)
w1 = []
for i in range(3):
    t = time.perf_counter(); s1.forward(p, bench.SIM_SEED, i); w1.append(time.perf_counter() - t)
step = statistics.mean(w1) - setup
full = mk(bench.T_STEPS)
t = time.perf_counter()
fw = full.forward(p, bench.SIM_SEED, 0)
wall = time.perf_counter() - t
print(json.dumps({
    "what": "reference simulate_forward, C3 1-h nowcast (120 steps), 1 core",
    **bench.host_info(), "full_hour_wall_s": wall, "rtf_full_hour": bench.SIM_SECONDS / wall,
    "extrapolated_from_1_step_s": setup + bench.T_STEPS * step, "setup_s": setup, "step_s": step,
    "cum_final_sum": float(fw["cum_per_step"][-1].sum()),
    "fnv_state": hex(fnv1a64_c(fw["link"], fw["pos"])),
    "kat_fnv_state": "0x5573a3f14223bbba"}), flush=True)
