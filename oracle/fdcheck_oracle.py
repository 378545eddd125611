"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Plain-Python restatement of the reference's FD-validation instrumentation
 on the compact per-agent state, for small cases:

* the instrumented engine_step (engine.cpp:70-125) with the traced relu / min /
  graft / carrier of SurrogateTrace (car_following.cpp:17-94) in record and
  replay mode and relaxed choices (soft_choices, node_model.cpp:21);
* the BranchTrace hash (branch_trace.hpp) in the reference's note order
  (engine.cpp:95,112; car_following.cpp:107,133,143-144,155;
  observation.cpp:15; node_model.cpp:23,50,87-90,168);
* run_gradcheck (pipeline.cpp:499-585).

Every arithmetic step is the reference's tensor operation on the same operands
in the same order, and exp/log are glibc's (Python's math), so results are
bit-identical to the reference.  The restatement is pinned against the
reference-generated fixtures tests/golden/f4_*.npz (tests/test_oracle_f4.py)
and is the specification the device probe engine (csrc/dtg_probe.cu) follows.
Records of a recording run are keyed by (step, agent) / (step, link), exactly
like the device; the reference consumes them in call order, which agrees on
the recorded control path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK = 0xFFFFFFFFFFFFFFFF
VALID = -1e-2        # kValidThreshold, car_following.hpp:12-13
ARRIVAL_TOL = 1e-2   # kArrivalTol, car_following.hpp:14-15
MASK_LARGE = 1e12    # kMaskLarge, car_following.hpp:16

FRACTIONAL, ZERO_ALPHA, OFF_PATH = 1, 2, 16


# ---- RngStream (rng.hpp:10-61) -----------------------------------------------------
def mix(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def fork(seed: int, label: int) -> int:
    return mix(seed ^ mix(label ^ 0x8E9B5C1D3A7F2406))


def bits(seed: int, a: int, b: int, c: int) -> int:
    h = mix(seed ^ mix(a))
    h = mix(h ^ mix(b ^ 0x6A09E667F3BCC909))
    return mix(h ^ mix(c ^ 0xBB67AE8584CAA73B))


def uniform(seed: int, a: int, b: int = 0, c: int = 0) -> float:
    return ((bits(seed, a, b, c) >> 11) + 0.5) * (1.0 / 9007199254740992.0)


def gumbel(seed: int, key: int, row: int, col: int) -> float:  # tensor.cpp:686-697
    return -math.log(-math.log(uniform(seed, key, row, col)))


# ---- BranchTrace (branch_trace.hpp) ------------------------------------------------
class BranchTrace:
    def __init__(self):
        self.h = 0xCBF29CE484222325

    def bit(self, b: bool):
        self.h = ((self.h ^ (0x9E if b else 0x7F)) * 0x100000001B3) & MASK

    def u64(self, v: int):
        for _ in range(8):
            self.h = ((self.h ^ (v & 0xFF)) * 0x100000001B3) & MASK
            v >>= 8


@dataclass
class Trace:
    """Keyed SurrogateTrace records of one recording run."""
    xp0: dict = field(default_factory=dict)     # (t, n) -> x'
    pk: dict = field(default_factory=dict)      # (t, n) -> (relu, min, cap) picks
    hard0: dict = field(default_factory=dict)   # (t, j) -> hard count
    soft0: dict = field(default_factory=dict)   # (t, j) -> soft count
    incpk: dict = field(default_factory=dict)   # (t, j) -> relu pick of q - qprev
    xbar0: dict = field(default_factory=dict)   # (t, n) -> position at transfer
    cnt0: dict = field(default_factory=dict)    # (t, j) -> agents on j
    na0: dict = field(default_factory=dict)     # t -> arrived agents
    recorded: bool = False


def two_softmax(V, g, kinv):
    """log_softmax -> y = (logz + g) / tau_g -> softmax, first argmax
    (node_model.cpp:13-25; tensor.cpp:407-433, 660-670) over live columns."""
    m = V[0]
    for x in V[1:]:
        m = max(m, x)
    z = 0.0
    for x in V:
        z += math.exp(x - m)
    lz = math.log(z) + m
    y = [((x - lz) + gg) * kinv for x, gg in zip(V, g)]
    m2 = y[0]
    for x in y[1:]:
        m2 = max(m2, x)
    z2 = 0.0
    for x in y:
        z2 += math.exp(x - m2)
    pi = [math.exp(x - m2) / z2 for x in y]
    best = 0
    for c in range(1, len(pi)):
        if pi[c] > pi[best]:
            best = c
    return pi, best


def simulate(net, link0, pos0, params, T, seed, noise_iteration, *, delta_n=1, tau=1.0, M=99999.0,
             gumbel_tau=0.01, tg=True, soft=False, sur=0, trace: Trace = None, trace_branches=True):
    """One instrumented simulate_forward (engine.cpp:227-254).  net = (succ_off,
    succ, length); params = [u, kappa, beta, alpha, cost]; sur: 0 none,
    1 record into `trace`, 2 replay from it.  Returns dict(cum_per_step, link,
    pos, hash, flags)."""
    succ_off, succ, length = ([int(x) for x in net[0]], [int(x) for x in net[1]],
                              [float(x) for x in net[2]])
    L, N = len(length), len(link0)
    u, kap, beta, alpha, cost = (list(map(float, a)) for a in params)
    dt = tau * delta_n
    kinv = 1.0 / gumbel_tau
    sim = fork(fork(seed, 7), noise_iteration)  # engine.cpp:49
    s_link, s_merge = fork(sim, 3), fork(sim, 4)
    lnk = [int(x) for x in link0]
    pos = [float(x) for x in pos0]
    record, replay = sur == 1, sur == 2
    bt = BranchTrace()
    flags = 0
    # initial_counts (engine.cpp:127-135)
    qprev = [0.0] * L
    for j in range(L):
        o = 0.5 * length[j]
        c = 0.0
        for n in range(N):
            if lnk[n] == j:
                c += (1.0 if pos[n] >= o else 0.0) * 1.0
        qprev[j] = c
    cum = [0.0] * L
    cum_hist = np.zeros((T, L))
    for t in range(T):
        on = [[] for _ in range(L)]
        for n in range(N):  # ascending agent id (engine.cpp:77-82)
            if lnk[n] >= 0:
                on[lnk[n]].append(n)
        x1 = list(pos)
        q = [0.0] * L
        for j in range(L):
            ids = on[j]
            m = len(ids)
            if record:
                trace.cnt0[(t, j)] = m
            elif replay and trace.cnt0.get((t, j)) != m:
                flags |= OFF_PATH
            if m == 0:
                continue
            # headways (car_following.cpp:96-126): stable argsort, descending
            order = sorted(range(m), key=lambda k: -pos[ids[k]])
            hw = [0.0] * m
            for r, k in enumerate(order):
                hw[k] = M if r == 0 else pos[ids[order[r - 1]]] - pos[ids[k]]
            if trace_branches:
                for n in ids:
                    bt.u64(n * L + j)
                for _ in ids:
                    bt.bit(True)
                for k in order:
                    bt.u64(k)
            dxf = (1.0 * u[j]) * dt
            jam = float(delta_n) / kap[j]
            Lj = length[j]
            bits_gap, bits_cong, bits_cap = [], [], []
            for k, n in enumerate(ids):
                x = pos[n]
                gap = hw[k] - jam
                if replay:
                    p1, p2, p3 = trace.pk[(t, n)]
                    a1, a2, a3 = (1.0 if p1 else 0.0), (1.0 if p2 else 0.0), (1.0 if p3 else 0.0)
                    dxc = (gap * a1 + 0.0 * (1.0 - a1)) * 1.0
                    dx = dxc * a2 + dxf * (1.0 - a2)
                    xp = x + dx
                    limit = (xp - trace.xp0[(t, n)]) + Lj if tg else Lj
                    xo = xp * a3 + limit * (1.0 - a3)
                else:
                    dxc = (gap if gap >= 0.0 else 0.0) * 1.0
                    dx = dxc if dxc <= dxf else dxf
                    xp = x + dx
                    limit = Lj
                    xo = xp if xp <= limit else limit
                    if record:
                        trace.pk[(t, n)] = (gap >= 0.0, dxc <= dxf, xp <= limit)
                        trace.xp0[(t, n)] = xp
                bits_gap.append(gap <= 0.0)
                bits_cong.append(dxc <= dxf)
                bits_cap.append(xp <= limit)
                x1[n] = xo
            if trace_branches and not sur:
                for b in bits_gap + bits_cong + bits_cap:
                    bt.bit(b)
            # midpoint_count (observation.cpp:9-20)
            o, sc = 0.5 * Lj, 5.0 / Lj
            hard = soft_sum = 0.0
            for n in ids:
                hard += (1.0 if x1[n] >= o else 0.0) * 1.0
            if trace_branches:
                for n in ids:
                    bt.bit(x1[n] >= o)
            if sur:
                for n in ids:
                    z = (x1[n] + (-o)) * sc
                    sg = 1.0 / (1.0 + math.exp(-z)) if z >= 0.0 else math.exp(z) / (1.0 + math.exp(z))
                    soft_sum += sg * 1.0
            if record:
                trace.hard0[(t, j)] = hard
                trace.soft0[(t, j)] = soft_sum
            q[j] = (soft_sum - trace.soft0[(t, j)]) + trace.hard0[(t, j)] if replay else hard
        # inc / cum (engine.cpp:109-113)
        incb = []
        for j in range(L):
            a = q[j] - qprev[j]
            if replay:
                pa = 1.0 if trace.incpk[(t, j)] else 0.0
                inc = a * pa + 0.0 * (1.0 - pa)
            else:
                inc = a if a >= 0.0 else 0.0
                if record:
                    trace.incpk[(t, j)] = a >= 0.0
            cum[j] = cum[j] + inc
            qprev[j] = q[j]
            incb.append(inc != 0.0)
        cum_hist[t] = cum
        if trace_branches and not sur:
            for b in incb:
                bt.bit(b)
        # node_step (node_model.cpp:151-181)
        arr = [n for n in range(N) if lnk[n] >= 0 and x1[n] >= VALID and x1[n] >= length[lnk[n]] - ARRIVAL_TOL]
        if record:
            trace.na0[t] = len(arr)
        elif replay and trace.na0.get(t) != len(arr):
            flags |= OFF_PATH
        for n in range(N):
            if lnk[n] >= 0:
                pos[n] = x1[n]
        if not arr:
            continue
        vac = []
        for j in range(L):  # vacancy_from_state (node_model.cpp:27-41)
            mn = M
            for n in on[j]:
                if x1[n] >= VALID and x1[n] < mn:
                    mn = x1[n]
            vac.append(mn > float(delta_n) / kap[j])
        nA = len(arr)
        lch = [-1] * nA
        cands = [[] for _ in range(L)]
        for r, n in enumerate(arr):  # link_choice (node_model.cpp:45-97)
            c = lnk[n]
            sj = list(succ[succ_off[c]:succ_off[c + 1]])
            if record:
                trace.xbar0[(t, n)] = x1[n]
            if sj:
                V = [1.0 * (beta[j] / cost[j]) - 0.0 for j in sj]
                g = [gumbel(s_link, t, n, j) for j in sj]
                pi, best = two_softmax(V, g, kinv)
                lch[r] = sj[best]
                for e, j in enumerate(sj):
                    lv = pi[e] * (1.0 if vac[j] else 0.0) if soft else (1.0 if e == best else 0.0) * (
                        1.0 if vac[j] else 0.0)
                    if lv != 0.0 and lv != 1.0:
                        flags |= FRACTIONAL
                    if lv == 1.0:
                        cands[j].append(r)
            elif trace_branches and not soft:
                V = [0.0 - MASK_LARGE] * L
                _, lch[r] = two_softmax(V, [gumbel(s_link, t, n, j) for j in range(L)], kinv)
        mwin = [-1] * L
        for i in range(L):  # merge_choice (node_model.cpp:99-120) + transfer (:122-149)
            ci = cands[i]
            if ci:
                V = []
                for r in ci:
                    prio = alpha[lnk[arr[r]]]
                    if prio == 0.0:
                        flags |= ZERO_ALPHA
                    V.append(1.0 * prio - 0.0)
                pi, w = two_softmax(V, [gumbel(s_merge, t, i, arr[r]) for r in ci], kinv)
                if soft and any(p != 0.0 and p != 1.0 for p in pi):
                    flags |= FRACTIONAL
                mwin[i] = ci[w]
            elif trace_branches and not soft:
                _, mwin[i] = two_softmax([0.0 - MASK_LARGE] * nA, [gumbel(s_merge, t, i, n) for n in arr], kinv)
        if trace_branches:
            for n in arr:
                bt.u64(n)
            for n in arr:
                for j in range(L):
                    bt.bit(j == lnk[n])
            if not soft:
                for r in range(nA):
                    for j in range(L):
                        bt.bit(j == lch[r])
            for _ in arr:
                bt.bit(True)
            for j in range(L):
                bt.bit(vac[j])
            for n in arr:
                bt.bit(succ_off[lnk[n] + 1] > succ_off[lnk[n]])
            if not soft:
                for i in range(L):
                    for r in range(nA):
                        bt.bit(r == mwin[i])
        for i in range(L):
            if mwin[i] >= 0 and cands[i]:
                n = arr[mwin[i]]
                entry = M
                if tg and replay:
                    entry = (x1[n] - trace.xbar0[(t, n)]) + M
                npos = ((-M) * 1.0 + 0.0 * (-M)) + 1.0 * entry
                pos[n] = npos
                lnk[n] = i if npos >= VALID else -1
    if record:
        trace.recorded = True
    return dict(cum_per_step=cum_hist, link=np.array(lnk, np.int32), pos=np.array(pos),
                hash=bt.h if trace_branches else 0xCBF29CE484222325, flags=flags)


# ---- run_gradcheck (pipeline.cpp:486-585) -----------------------------------------
def chain_network(n_phys=3, link_len=300.0, inflow_len=100.0):
    """make_chain_network (pipeline.cpp:486-496): (frm, to, length, kind, n_nodes)."""
    frm = [n_phys + 1] + list(range(n_phys)) + [n_phys]
    to = [0] + list(range(1, n_phys + 1)) + [n_phys + 2]
    ln = [inflow_len] + [link_len] * n_phys + [inflow_len]
    kind = [1] + [0] * n_phys + [2]
    return (np.array(frm, np.int32), np.array(to, np.int32), np.array(ln), np.array(kind, np.int32), n_phys + 3)


def chain_seed(length, agents, delta_n=1, seeding_kappa=0.2):
    """seed_agents (engine.cpp:156-189) on a network with one inflow link (0)."""
    spacing = delta_n / seeding_kappa
    pos = [length[0] - a * spacing for a in range(agents)]
    if pos and pos[-1] < 0.0:
        raise RuntimeError("inflow queue does not fit")
    return np.zeros(agents, np.int32), np.array(pos)


def gradcheck_params(seed, attempt, L):
    """pipeline.cpp:512-520."""
    pr = fork(seed, 9000 + attempt)
    rng = [(13.9, 22.2), (0.18, 0.22), (0.0, 5.0), (0.01, 5.0), (0.5, 2.0)]
    return [np.array([lo + (hi - lo) * uniform(pr, b, l) for l in range(L)]) for b, (lo, hi) in enumerate(rng)]


def run_gradcheck(port_lib, draws=20, steps=20, agents=5, tol=1e-4, seed=1):
    """run_gradcheck restated: the adjoint from the C port (oracle/dtsim_port.c,
    hard choices == relaxed choices on the chain: every row is one-hot) and the
    central differences from `simulate` in surrogate replay."""
    from oracle.oracle import Params, PortScenario, csr_from_links

    frm, to, ln, kind, _ = chain_network()
    L = len(ln)
    succ_off, succ = csr_from_links(frm, to)
    link0, pos0 = chain_seed(ln, agents)
    port = PortScenario(port_lib, frm, to, ln, link0=link0, pos0=pos0, horizon_steps=steps, obs_interval_s=steps)
    net = (succ_off, succ, ln)
    rep = dict(max_rel_err=0.0, draws=draws, redraws=0, passed=False, per_draw_max=[])
    attempt = 0
    for _ in range(draws):
        clean, draw_max, tries = False, 0.0, 0
        while tries < 60 and not clean:
            p = gradcheck_params(seed, attempt, L)
            attempt += 1
            g = port.gradient(Params(*p), seed, 0, wc=np.ones(L))["grads"]
            tr = Trace()
            base = simulate(net, link0, pos0, p, steps, seed, 0, soft=True, sur=1, trace=tr)
            clean, draw_max = True, 0.0
            for b in range(5):
                for l in range(L):
                    x0 = p[b][l]
                    h = 1e-5 * max(1.0, abs(x0))
                    f = []
                    for sgn in (1.0, -1.0):
                        q = [a.copy() for a in p]
                        q[b][l] = x0 + sgn * h
                        r = simulate(net, link0, pos0, q, steps, seed, 0, soft=True, sur=2, trace=tr)
                        ok = r["hash"] == base["hash"] and not (r["flags"] & OFF_PATH)
                        s = 0.0
                        for v in r["cum_per_step"][-1]:
                            s += v
                        f.append((ok, s))
                    if not (f[0][0] and f[1][0]):
                        clean = False
                        break
                    fd = (f[0][1] - f[1][1]) / (2.0 * h)
                    abs_err = abs(g[b][l] - fd)
                    if abs_err < 1e-6:
                        continue
                    draw_max = max(draw_max, abs_err / max(abs(g[b][l]), abs(fd)))
                if not clean:
                    break
            tries += 1
            rep["redraws"] += 1
        if not clean:
            raise RuntimeError("gradcheck: could not find a kink-free parameter draw")
        rep["per_draw_max"].append(draw_max)
        rep["max_rel_err"] = max(rep["max_rel_err"], draw_max)
    rep["passed"] = rep["max_rel_err"] < tol
    return rep
