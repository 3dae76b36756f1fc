"""CPU oracle for the population-parallel NEAT hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline leg may import this module, and only as the
checker.  The product package (``paper_2404_01817_b200``) never imports it.

This is an independent restatement of the algorithm of the reference
``arrayneat`` 0.1.0 (``/root/reference/pkg/src/arrayneat``), written
genome-at-a-time with explicit loops instead of the reference's
population-wide NumPy masking.  Every function cites the reference lines it
restates.  It is pinned against golden vectors produced by running the
reference itself (``tests/golden/make_goldens.py`` -> ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks the pin).

Parity status: pinned for RNG, transform, forward, distance, crossover,
mutation, speciation, spawn allocation and reproduce (reference goldens).
The recurrent and HyperNEAT restatements (``recurrent_rollout``,
``substrate_fitness``) have no reference implementation, so their
parity is UNPINNED beyond the CPPN query, which is a plain forward pass.
"""

from __future__ import annotations

import math

import numpy as np

# -- genome layout (genome.py:29-35) -------------------------------------------
KEY, BIAS, RESP, AGG, ACT = range(5)
CIN, COUT, CEN, CW = range(4)

# -- function table (functions.py:20-39); code 4 (min) is the builder's
# extension required by north_star (no reference oracle for it) ------------------


def act_apply(code: int, x: np.ndarray) -> np.ndarray:
    """Activation table, functions.py:26-31 (sigmoid = exp(-logaddexp(0,-x)), :20-22)."""
    if code == 0:
        return x
    if code == 1:
        return np.tanh(x)
    if code == 2:
        return np.exp(-np.logaddexp(0.0, -x))
    if code == 3:
        return np.maximum(x, 0.0)
    raise ValueError(f"unknown activation code {code}")


def agg_apply(code: int, terms: list[np.ndarray], batch: int) -> np.ndarray:
    """Aggregation table, functions.py:34-39; empty set -> 0 (inference.py:238-240)."""
    if not terms:
        return np.zeros(batch)
    stack = np.stack(terms, axis=-1)
    if code == 0:
        return stack.sum(axis=-1)
    if code == 1:
        return stack.prod(axis=-1)
    if code == 2:
        return stack.max(axis=-1)
    if code == 3:
        return stack.sum(axis=-1) / stack.shape[-1]
    if code == 4:
        return stack.min(axis=-1)
    raise ValueError(f"unknown aggregation code {code}")


# -- counter-based RNG (rng.py) ---------------------------------------------------
_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB


def mix64(z: int) -> int:
    """splitmix64 finaliser on a Python int, rng.py:25-29."""
    z &= _M64
    z = ((z ^ (z >> 30)) * MIX1) & _M64
    z = ((z ^ (z >> 27)) * MIX2) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, *path: int) -> int:
    """Key of RngStream(seed, path) for scalar tokens, rng.py:56-69 and _fold :32-34.

    Tokens are two's complement 64-bit (rng.py:37-42)."""
    key = mix64(seed & _M64)
    for tok in path:
        key = mix64(key ^ mix64((int(tok) & _M64) + GOLDEN))
    return key


def raw_draw(key: int, j: int) -> int:
    """j-th raw value (0-based) of a stream: mix64(key + (j+1)*G), rng.py:86-90."""
    return mix64(int(key) + ((int(j) + 1) * GOLDEN & _M64))


def bits_to_uniform(bits: int) -> float:
    """((bits >> 11) + 0.5) * 2^-53, exact in float64, rng.py:96."""
    return ((bits >> 11) + 0.5) * 2.0 ** -53


class Stream:
    """Scalar restatement of one RngStream: key + counter, rng.py:45-134."""

    def __init__(self, key: int):
        self.key = key
        self.counter = 0

    def uniforms(self, n: int) -> np.ndarray:
        out = np.array([bits_to_uniform(raw_draw(self.key, self.counter + j)) for j in range(n)])
        self.counter += n
        return out

    def normals(self, n: int) -> np.ndarray:
        """Box-Muller with u1 = first n draws, u2 = next n, rng.py:99-105."""
        u = self.uniforms(2 * n)
        return np.sqrt(-2.0 * np.log(u[:n])) * np.cos(2.0 * np.pi * u[n:])

    def uniform_cell(self, base: int, col: int) -> float:
        return bits_to_uniform(raw_draw(self.key, base + col))

    def normal_cell(self, base: int, width: int, col: int) -> float:
        """normals_at cell (rng.py:125-134): u1 at base+col, u2 at base+width+col."""
        u1 = self.uniform_cell(base, col)
        u2 = self.uniform_cell(base, width + col)
        return float(np.sqrt(-2.0 * np.log(np.float64(u1))) * np.cos(2.0 * np.pi * np.float64(u2)))

    def skip(self, n: int) -> int:
        base = self.counter
        self.counter += n
        return base


# -- transform (inference.py:82-147) ----------------------------------------------


def live_rows(nodes: np.ndarray) -> list[int]:
    return [r for r in range(nodes.shape[0]) if not math.isnan(nodes[r, KEY])]


def key_to_row(nodes: np.ndarray) -> dict[int, int]:
    """Exact key -> row map (search.py:103-124 resolves the same rows)."""
    return {int(nodes[r, KEY]): r for r in live_rows(nodes)}


def enabled_edges(nodes: np.ndarray, conns: np.ndarray) -> list[tuple[int, int, float, int]]:
    """(src_row, dst_row, weight, conn_row) of live & enabled conns, inference.py:93-112."""
    rows = key_to_row(nodes)
    out = []
    for c in range(conns.shape[0]):
        if math.isnan(conns[c, CIN]) or conns[c, CEN] != 1.0:
            continue
        out.append((rows[int(conns[c, CIN])], rows[int(conns[c, COUT])], float(conns[c, CW]), c))
    return out


def transform_genome(nodes: np.ndarray, conns: np.ndarray, num_inputs: int, num_outputs: int) -> dict:
    """Kahn order with the smallest ready ROW first, one node per step
    (inference.py:114-141); cyclic if live nodes remain (:143).

    Repeated (in, out) pairs follow the reference exactly: the dense incoming
    row keeps the LAST conn row's weight (fancy assignment, :108-112), the
    indegree counts every row (np.add.at, :114-115), and a picked source
    decrements its successor once per distinct successor when max_nodes <= 64
    (bitmask OR, :116-122,136-137) but once per row above that
    (np.subtract.at, :139-141) -- so with <= 64 rows a repeated pair leaves its
    destination unready and the genome reads as cyclic."""
    rows = key_to_row(nodes)
    rows_edges = enabled_edges(nodes, conns)
    last: dict[tuple[int, int], tuple[int, int, float, int]] = {}
    for e in rows_edges:
        last[(e[0], e[1])] = e
    edges = sorted(last.values(), key=lambda e: e[3])
    bitmask = nodes.shape[0] <= 64
    indeg = {r: 0 for r in rows.values()}
    succ: dict[int, list[int]] = {r: [] for r in rows.values()}
    for s, d, _, _ in rows_edges:
        indeg[d] += 1
        if not (bitmask and d in succ[s]):
            succ[s].append(d)
    remaining = set(rows.values())
    order: list[int] = []
    while True:
        ready = [r for r in remaining if indeg[r] == 0]
        if not ready:
            break
        pick = min(ready)
        order.append(pick)
        remaining.discard(pick)
        for d in succ[pick]:
            indeg[d] -= 1
    return {
        "order": order,
        "edges": edges,
        "input_rows": [rows[k] for k in range(num_inputs)],
        "output_rows": [rows[k] for k in range(num_inputs, num_inputs + num_outputs)],
        "cyclic": bool(remaining),
    }


def order_array(tr: dict, n: int) -> np.ndarray:
    """(n,) float64 NaN-padded order as StackedNetworks.order stores it (inference.py:125,133)."""
    out = np.full(n, np.nan)
    out[: len(tr["order"])] = tr["order"]
    return out


def incoming_dense(tr: dict, n: int) -> np.ndarray:
    """(n, n) incoming[dst, src] = weight, NaN elsewhere (inference.py:108-112)."""
    inc = np.full((n, n), np.nan)
    for s, d, w, _ in tr["edges"]:
        inc[d, s] = w
    return inc


# -- forward (inference.py:185-262) -------------------------------------------------


def forward_genome(nodes: np.ndarray, tr: dict, inputs: np.ndarray) -> np.ndarray:
    """inputs (B, I) float64 -> (B, O): input rows hold raw inputs and are never
    activated (inference.py:200-215); node = act(bias + response * agg(w * v))
    (:242-253), empty aggregation = 0 (:238-240)."""
    inputs = np.asarray(inputs, dtype=np.float64)
    batch = inputs.shape[0]
    value: dict[int, np.ndarray] = {}
    input_rows = set(tr["input_rows"])
    for i, r in enumerate(tr["input_rows"]):
        value[r] = inputs[:, i]
    into: dict[int, list[tuple[int, float]]] = {}
    for s, d, w, _ in tr["edges"]:
        into.setdefault(d, []).append((s, w))
    for r in tr["order"]:
        if r in input_rows:
            continue
        terms = [w * value[s] for s, w in sorted(into.get(r, []))]
        agg = agg_apply(int(nodes[r, AGG]), terms, batch)
        value[r] = act_apply(int(nodes[r, ACT]), nodes[r, BIAS] + nodes[r, RESP] * agg)
    return np.stack([value[r] for r in tr["output_rows"]], axis=-1)


def forward_population(nodes: np.ndarray, conns: np.ndarray, inputs: np.ndarray,
                       num_inputs: int, num_outputs: int) -> np.ndarray:
    """(P,N,5),(P,C,4),(P,B,I) -> (P,B,O), genome by genome."""
    out = []
    for p in range(nodes.shape[0]):
        tr = transform_genome(nodes[p], conns[p], num_inputs, num_outputs)
        if tr["cyclic"]:
            raise ValueError(f"genome {p} is cyclic")
        out.append(forward_genome(nodes[p], tr, inputs[p]))
    return np.stack(out)


# -- fitness (problems.py:54-61) ------------------------------------------------------
XOR_IN = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 0.0], [1.0, 1.0]])
XOR_OUT = np.array([0.0, 1.0, 1.0, 0.0])


def xor_fitness(outputs: np.ndarray) -> float:
    """4 - sum of squared errors over the four cases, problems.py:54-56."""
    return float(4.0 - np.sum((outputs.reshape(4) - XOR_OUT) ** 2))


def regression_fitness(outputs: np.ndarray, targets: np.ndarray) -> float:
    """-MSE, problems.py:59-61."""
    return float(-np.mean((outputs.reshape(-1) - targets) ** 2))


# -- distance (evolution.py:425-488) -----------------------------------------------------


def distance_genome(n1: np.ndarray, c1: np.ndarray, n2: np.ndarray, c2: np.ndarray,
                    c_disjoint: float, c_homologous: float) -> float:
    """Compatibility distance; homologous terms summed sequentially in genome-1
    row order (nodes, then conns) as np.bincount does (evolution.py:466,477)."""
    k2 = {int(n2[r, KEY]): r for r in live_rows(n2)}
    p2 = {}
    for r in range(c2.shape[0]):
        if not math.isnan(c2[r, CIN]):
            p2[(int(c2[r, CIN]), int(c2[r, COUT]))] = r
    rows1 = live_rows(n1)
    node_sum = 0.0
    node_hom = 0
    for r in rows1:
        o = k2.get(int(n1[r, KEY]))
        if o is None:
            continue
        node_hom += 1
        node_sum += (abs(n1[r, BIAS] - n2[o, BIAS]) + abs(n1[r, RESP] - n2[o, RESP])
                     + float(n1[r, AGG] != n2[o, AGG]) + float(n1[r, ACT] != n2[o, ACT])) / 4.0
    crows1 = [r for r in range(c1.shape[0]) if not math.isnan(c1[r, CIN])]
    conn_sum = 0.0
    conn_hom = 0
    for r in crows1:
        o = p2.get((int(c1[r, CIN]), int(c1[r, COUT])))
        if o is None:
            continue
        conn_hom += 1
        conn_sum += (abs(c1[r, CW] - c2[o, CW]) + abs(c1[r, CEN] - c2[o, CEN])) / 2.0
    disjoint = (len(rows1) - node_hom) + (len(k2) - node_hom) \
        + (len(crows1) - conn_hom) + (len(p2) - conn_hom)
    hom = node_hom + conn_hom
    attr = (node_sum + conn_sum) / hom if hom > 0 else 0.0
    total = max(len(rows1) + len(crows1), len(k2) + len(p2))
    return c_disjoint * disjoint / total + c_homologous * attr


# -- synthetic config-2 population ----------------------------------------


def synthetic_population(pop: int, max_nodes: int, max_conns: int, num_inputs: int,
                         num_outputs: int, seed: int = 20261018, variant: str = "T",
                         min_conns: int = 256, max_conns_drawn: int = 512,
                         max_hidden: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """SURVEY.md §8d generator: io keys at rows 0..io-1, H~U{0..Hmax} hidden nodes
    with distinct random keys at random rows, E~U{min..max} acyclic conns
    (src not output, dst not input, random topological rank) at random rows,
    enabled~Bern(0.9), weight/bias~N(0,1), response 1; variant "T" = tanh/sum,
    "M" = act, agg ~ U{0..3}."""
    rng = np.random.default_rng(seed)
    io = num_inputs + num_outputs
    hmax = max_nodes - io if max_hidden is None else min(max_hidden, max_nodes - io)
    nodes = np.full((pop, max_nodes, 5), np.nan)
    conns = np.full((pop, max_conns, 4), np.nan)
    for p in range(pop):
        h = int(rng.integers(0, hmax + 1))
        hidden_keys = io + rng.choice(2 ** 20, size=h, replace=False)
        hidden_rows = io + rng.choice(max_nodes - io, size=h, replace=False)
        nkeys = np.concatenate([np.arange(io), hidden_keys]).astype(np.float64)
        nrows = np.concatenate([np.arange(io), hidden_rows])
        nn = nkeys.size
        nodes[p, nrows, KEY] = nkeys
        nodes[p, nrows, BIAS] = np.clip(rng.standard_normal(nn), -30, 30)
        nodes[p, nrows, RESP] = 1.0
        if variant == "M":
            nodes[p, nrows, AGG] = rng.integers(0, 4, nn)
            nodes[p, nrows, ACT] = rng.integers(0, 4, nn)
        else:
            nodes[p, nrows, AGG] = 0.0
            nodes[p, nrows, ACT] = 1.0
        # topological rank: inputs first, then a random permutation of the rest
        rank = np.empty(nn)
        rank[:num_inputs] = -1.0
        rank[num_inputs:] = rng.permutation(nn - num_inputs)
        is_out = (nkeys >= num_inputs) & (nkeys < io)
        is_in = nkeys < num_inputs
        src_ok = ~is_out
        dst_ok = ~is_in
        cand = np.argwhere(src_ok[:, None] & dst_ok[None, :] & (rank[:, None] < rank[None, :]))
        e = min(int(rng.integers(min_conns, max_conns_drawn + 1)), cand.shape[0], max_conns)
        pick = cand[rng.choice(cand.shape[0], size=e, replace=False)]
        crow = rng.choice(max_conns, size=e, replace=False)
        conns[p, crow, CIN] = nkeys[pick[:, 0]]
        conns[p, crow, COUT] = nkeys[pick[:, 1]]
        conns[p, crow, CEN] = (rng.random(e) < 0.9).astype(np.float64)
        conns[p, crow, CW] = np.clip(rng.standard_normal(e), -30, 30)
    return nodes, conns


# -- HyperNEAT restatement (no reference: SPEC.md:8; parity UNPINNED beyond the
# CPPN query, which is forward_genome on coordinate inputs) ----------------------


def substrate_query_inputs(grid: int = 8) -> np.ndarray:
    """q = k*n + j -> (x_j, y_j, x_k, y_k) on an grid x grid lattice over [-1,1]^2."""
    lin = np.linspace(-1.0, 1.0, grid)
    pts = [(lin[c], lin[r]) for r in range(grid) for c in range(grid)]
    n = len(pts)
    return np.array([[pts[j][0], pts[j][1], pts[k][0], pts[k][1]] for k in range(n) for j in range(n)])


def substrate_fitness(nodes: np.ndarray, conns: np.ndarray, x: np.ndarray, t: np.ndarray) -> float:
    """W = CPPN(queries) (forward_genome, float64); fitness = -mean((tanh(X W^T) - t)^2)."""
    tr = transform_genome(nodes, conns, 4, 1)
    q = substrate_query_inputs()
    w = forward_genome(nodes, tr, q)[:, 0].reshape(64, 64)
    y = np.tanh(x.astype(np.float64) @ w.T)
    return float(-np.mean((y - t.astype(np.float64)[:, None]) ** 2))


# -- recurrent restatement (no reference: SPEC.md:360 rejects recurrent
# genomes; parity UNPINNED) -------------------------------------------------------


def recurrent_rollout(nodes: np.ndarray, conns: np.ndarray, num_inputs: int, num_outputs: int,
                      a: np.ndarray, m: np.ndarray, s0: np.ndarray, steps: int, sweeps: int) -> float:
    """K synchronous sweeps per environment step over the enabled graph
    (cycles allowed), node math of inference.py:217-253; s' = tanh(A s + M a)."""
    rows = key_to_row(nodes)
    into: dict[int, list[tuple[int, float]]] = {}
    for s_, d_, w_, _ in enabled_edges(nodes, conns):
        into.setdefault(d_, []).append((s_, w_))
    in_rows = [rows[k] for k in range(num_inputs)]
    out_rows = [rows[k] for k in range(num_inputs, num_inputs + num_outputs)]
    hidden = [r for r in live_rows(nodes) if r not in set(in_rows)]
    v = {r: 0.0 for r in live_rows(nodes)}
    s = np.asarray(s0, dtype=np.float64).copy()
    reward = 0.0
    for _ in range(steps):
        reward += float(s[0])
        for i, r in enumerate(in_rows):
            v[r] = float(s[i]) if i < s.size else 0.0
        for _ in range(sweeps):
            new = {}
            for r in hidden:
                terms = [np.array([w * v[src]]) for src, w in sorted(into.get(r, []))]
                agg = agg_apply(int(nodes[r, AGG]), terms, 1)[0]
                new[r] = float(act_apply(int(nodes[r, ACT]), np.array([nodes[r, BIAS] + nodes[r, RESP] * agg]))[0])
            v.update(new)
        act = np.array([v[r] for r in out_rows])
        s = np.tanh(a @ s + m @ act)
    return reward


# -- cart-pole episode replay (problems.py:107-177), test infrastructure only ---------


def _two_prod(a: float, b: float) -> tuple[float, float]:
    """Exact a*b = p + e (Dekker split; equals the device's fma(a, b, -p))."""
    p = a * b
    sp = 134217729.0  # 2^27 + 1
    ta = sp * a
    ah = ta - (ta - a)
    al = a - ah
    tb = sp * b
    bh = tb - (tb - b)
    bl = b - bh
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def _dd_two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _dd_add(a, b):
    s, e = _dd_two_sum(a[0], b[0])
    return _dd_two_sum(s, e + (a[1] + b[1]))


def _dd_mul(a, b):
    p, e = _two_prod(a[0], b[0])
    return _dd_two_sum(p, e + (a[0] * b[1] + a[1] * b[0]))


def cos_sin_device(x: float) -> tuple[float, float]:
    """Bitwise restatement of the cart-pole kernel's double-double cos/sin
    (csrc/forward.cu cos_sin_cr), for |x| <= 0.5."""
    from fractions import Fraction
    fh, fl = [], []
    for n in range(20):
        f = Fraction(1, math.factorial(n))
        fh.append(float(f))
        fl.append(float(f - Fraction(float(f))))
    x2h = x * x
    y = _two_prod(x, x)
    assert y[0] == x2h

    def series(j0):
        acc = (0.0, 0.0)
        for k in range(8, -1, -1):
            n = j0 + 2 * k
            c = (-fh[n], -fl[n]) if k & 1 else (fh[n], fl[n])
            acc = _dd_add(_dd_mul(acc, y), c)
        return acc
    cs = series(0)
    sn = _dd_mul(series(1), (x, 0.0))
    return cs[0] + cs[1], sn[0] + sn[1]


def cartpole_episode(nodes: np.ndarray, conns: np.ndarray, start, cos_sin=None, max_steps: int = 500) -> int:
    """Steps survived by one genome (problems.py:138-177 lockstep semantics:
    Euler step, bang-bang force sign(output > 0), termination |x| > 2.4 or
    |theta| > 12 deg).  ``cos_sin`` picks the libm: None = numpy's (the
    reference), ``cos_sin_device`` = the kernel's."""
    tr = transform_genome(nodes, conns, 4, 1)
    g, mc, mp, hl, fm, dt = 9.8, 1.0, 0.1, 0.5, 10.0, 0.02
    tm, pl = mc + mp, mp * hl
    x, xd, th, thd = (float(v) for v in start)
    steps = 0
    for _ in range(max_steps):
        out = forward_genome(nodes, tr, np.array([[x, xd, th, thd]]))[0, 0]
        force = fm if out > 0 else -fm
        if cos_sin is None or abs(th) > 0.5:
            ct, st = float(np.cos(th)), float(np.sin(th))
        else:
            ct, st = cos_sin(th)
        tmp = (force + pl * thd ** 2 * st) / tm
        tacc = (g * st - ct * tmp) / (hl * (4.0 / 3.0 - mp * ct ** 2 / tm))
        xacc = tmp - pl * tacc * ct / tm
        x, xd, th, thd = x + dt * xd, xd + dt * xacc, th + dt * thd, thd + dt * tacc
        steps += 1
        if abs(x) > 2.4 or abs(th) > 12 * 2 * math.pi / 360:
            break
    return steps
