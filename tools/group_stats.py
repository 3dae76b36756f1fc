"""Program statistics of the config-2 population: groups, sizes, rounds."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2404_01817_b200 as tn
from paper_2404_01817_b200.synthetic import synthetic_population
n, c = synthetic_population(1000, 128, 512, 32, 8, seed=20261018)
st, _ = tn.transform_arrays(n, c, 32, 8)
prog = st.program.cpu().numpy()
from paper_2404_01817_b200 import _native
L_groups = 48  # off_groups for O=8: align16(32+16)=48
hdr = prog[:, :32].view(np.int32)
ng = hdr[:, 7]; steps = hdr[:, 0]; edges = hdr[:, 1]; slots = hdr[:, 2]
sizes = []; rounds = []; cls = []
for p in range(1000):
    g = prog[p, 48:48 + 16 * ng[p]].reshape(-1, 16)
    sizes += list(g[:, 0]); cls += list(g[:, 1]); rounds += list(g[:, 2:4].copy().view(np.uint16)[:, 0])
sizes = np.array(sizes); rounds = np.array(rounds)
print("groups/genome", ng.mean(), "steps", steps.mean(), "edge entries", edges.mean(), "slots", slots.mean())
print("group size hist", np.bincount(sizes))
print("rounds mean", rounds.mean(), "hist", np.bincount(np.minimum(rounds, 40))[:41])
print("edge-slots per genome (sum gw*rounds)", (np.where(sizes==3,4,sizes)*rounds).sum()/1000)
cnts = []
for p in range(1000):
    g = prog[p, 48:48 + 16 * ng[p]].reshape(-1, 16)
    cnts.append(g[:, 8:16].copy().view(np.uint16).astype(np.int64).sum())
print("real entries / genome", np.mean(cnts), "padding frac", 1 - np.sum(cnts) / (np.where(sizes==3,4,sizes)*rounds).sum())
lv = []
sp, _ = tn.transform_arrays(n, c, 32, 8, layout="split")
pr = sp.program.cpu().numpy()
hd = pr[:, :32].view(np.int32)
cin = []; ch = []
for p in range(1000):
    g = pr[p, 48:48 + 32 * hd[p, 7]].reshape(-1, 32)
    cin.append(g[:, 16:24].copy().view(np.uint16).astype(np.int64).sum())
    ch.append(g[:, 24:32].copy().view(np.uint16).astype(np.int64).sum())
print("input-sourced edges / genome", np.mean(cin), "hidden-sourced", np.mean(ch))
