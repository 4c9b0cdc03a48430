"""An independent brute-force execution simulator (test infrastructure).

It knows nothing about Algorithm 1's queue scan, Q_temp, offsets or
CheckExecuted.  It models the paper's execution semantics directly
(§4.2 "Initialization" and "Backward planning", §3 queue order):

  * every GPU (node n, stage s) keeps ALL backward intervals ever planned on it
    and the end of its last forward (forwards are FIFO per GPU);
  * a forward on stage s starts at max(end of the task's stage s-1 forward
    (its dispatch time for stage 1), end of the GPU's last forward) and is
    pushed past any planned backward interval it would overlap, until it fits;
  * a training task's backward runs stages S..1 in reverse, each starting at
    max(end of its previous backward stage, end of the GPU's latest backward);
  * inference tasks are dispatched at arrival; training task j is released at
    max(a_min_j, end of training task j-1's stage-1 forward); ties go to
    inference (the DESIGN.md reading R-19).

Placing a task on a node under these rules is the "one-step extension" used
to pin the oracle's planned paths and response times bitwise.
"""
from __future__ import annotations

import math


class Cluster:
    def __init__(self, N, S, eta_f, eta_b):
        self.N, self.S = N, S
        self.ef = list(map(float, eta_f))
        self.eb = list(map(float, eta_b))
        self.fwd_last = [[-math.inf] * S for _ in range(N)]
        self.bwd = [[[] for _ in range(S)] for _ in range(N)]

    def plan_forward(self, n, w, a):
        """Forward path of a task of weight w dispatched at a on node n (no commit)."""
        path = []
        e = a
        for s in range(self.S):
            d = self.ef[n * self.S + s] * w
            t = e if e >= self.fwd_last[n][s] else self.fwd_last[n][s]
            moved = True
            while moved:
                moved = False
                for (b0, b1) in self.bwd[n][s]:
                    if t < b1 and b0 < t + d:
                        t = b1
                        moved = True
            path.append((t, t + d))
            e = t + d
        return path

    def commit(self, n, w, path, train):
        for s in range(self.S):
            self.fwd_last[n][s] = path[s][1]
        if not train:
            return None
        back = [None] * self.S
        x = path[-1][1]
        for s in range(self.S - 1, -1, -1):
            latest = max((b1 for (_, b1) in self.bwd[n][s]), default=-math.inf)
            sb = x if x >= latest else latest
            eb = sb + self.eb[n * self.S + s] * w
            self.bwd[n][s].append((sb, eb))
            back[s] = (sb, eb)
            x = eb
        return back


def dispatch_order(arrival, lbk, n_inf, path_of):
    """Yield (task, dispatch_time) in global-queue order; path_of(task) must
    return the committed forward path of an already dispatched task."""
    nI = n_inf
    nT = len(arrival) - nI
    i = j = 0
    r = arrival[nI] if nT > 0 else math.inf
    while i < nI or j < nT:
        t_inf = arrival[i] if i < nI else math.inf
        if t_inf <= r:
            yield i, t_inf
            i += 1
        else:
            task = nI + j
            yield task, r
            j += 1
            if j < nT:
                s1_end = path_of(task)[0][1]
                amin = arrival[nI + j]
                r = s1_end if s1_end > amin else amin
            else:
                r = math.inf


def task_w(v):
    l = v & 0xFFF
    C = (v >> 12) & 0xFF
    return float(C * l * l)


def simulate_fixed(N, S, eta_f, eta_b, arrival, lbk, n_inf, placement, probe_all=False):
    """Run the trace with a forced placement.  Returns (paths, backs, probes)
    where probes[task][n] = R of the one-step extension on node n (if probe_all)."""
    cl = Cluster(N, S, eta_f, eta_b)
    paths = {}
    backs = {}
    probes = {}
    for task, a in dispatch_order(arrival, lbk, n_inf, lambda t: paths[t]):
        v = int(lbk[task])
        w = task_w(v)
        train = task >= n_inf
        if probe_all:
            probes[task] = [cl.plan_forward(n, w, a)[-1][1] - a for n in range(N)]
        n = int(placement[task])
        p = cl.plan_forward(n, w, a)
        paths[task] = p
        backs[task] = cl.commit(n, w, p, train)
    return paths, backs, probes
