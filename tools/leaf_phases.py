"""Phase timestamps (us, CTA 0) of the whole-leaf kernel on an m x 128 leaf (debug hook
tcqr_debug_leaf_timestamps); phases: load, then per op (panel: mgs, gram+barrier, sum, barrier,
chol+S, apply; proj: partial, owner sum, gather, update; tagged reductions), then the final write."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1912_05508_b200 as tq
import workloads as W
tq.init(0)
L = tq.lib()
L.tcqr_debug_leaf_timestamps.argtypes = [ctypes.c_void_p]
names = ["load"]
for op in ["P0", "J01", "P1", "J0123", "P2", "J23", "P3"]:
    if op[0] == "P":
        names += [op + s for s in (":mgs", ":publish", ":ownersum", ":gather", ":chol+S", ":apply+st")]
    else:
        names += [op + s for s in (":partial+pub", ":ownersum", ":gather", ":update")]
names += ["write"]
for m in [int(v) for v in (sys.argv[1:] or ["32768"])]:  # m <= 148 * 256 (leaf kernel)
    dbg = torch.zeros(128, dtype=torch.int64, device="cuda")
    A = W.gaussian_cuda(m, 128, 3)
    Q = torch.empty_like(A)
    R = torch.empty(128, 128, device="cuda").t()
    tq.set_config(use_graphs=0)
    for _ in range(3):
        tq.factor(A, Q, R)
    L.tcqr_debug_leaf_timestamps(ctypes.c_void_p(dbg.data_ptr()))
    runs, extra, probes, skew = [], [], [], []
    for _ in range(5):
        dbg.zero_()
        tq.factor(A, Q, R)
        torch.cuda.synchronize()
        d = dbg.cpu().numpy().astype(np.int64)
        runs.append(np.diff(d[:len(names) + 1]) / 1000.0)
        extra.append(((d[102] - d[100]) / 1000.0, (d[104] - d[102]) / 1000.0, (d[101] - d[100]) / 1000.0))
        probes.append(d[110:116].copy())
        # latest CTA's Gram publish minus CTA 0's, per panel (ops 0, 2, 4, 6; CTA 0 slots 3, 13, 23, 33)
        skew.append([(d[120 + o] - d[i]) / 1000.0 for o, i in zip((0, 2, 4, 6), (3, 13, 23, 33))])
    L.tcqr_debug_leaf_timestamps(None)
    med = np.median(np.array(runs), axis=0)
    print(f"m={m}: total {med.sum():.1f} us; last panel: chol {np.median([e[0] for e in extra]):.2f} us, "
          f"S + apply before stores {np.median([e[1] for e in extra]):.2f} us")
    pr = np.median(np.array(probes), axis=0)
    print("  MGS step 5 of panel 2, warp 0 (cycles): colbuf+dot %d, shfl %d, sqrt/rcp/rkj %d, "
          "R+q publish %d, update %d, column publish %d" % tuple(pr))
    print("  latest CTA publish - CTA 0 publish per panel (us):", np.round(np.median(np.array(skew), axis=0), 2))
    for nm, v in zip(names, med):
        print(f"  {nm:16s} {v:7.2f}")
