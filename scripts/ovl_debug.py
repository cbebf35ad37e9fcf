import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_1910_11110_b200 as coh
from paper_1910_11110_b200.overlap import Registry, gen_workload
from make_golden_overlap import ref_closure
ctx = coh.Context(0)
views, modes, off = gen_workload(100, 8, 256, 600, 3000, 5, n_scalars=4, max_view_len=32, p_same_site=0.8)
reg = Registry(ctx, views)
out, cnt, st = reg.closure(modes, off)
w_out, w_cnt, w_st = ref_closure(views, modes, off)
bad = np.nonzero(st != w_st)[0]
print("bad", len(bad), "of", len(st))
for b in bad[:5]:
    print("block", b, "got", st[b], "want", w_st[b])
    for m in modes[off[b]:off[b+1]]:
        v = views[m["var"]] if m["flags"] & 1 else None
        print("   mode", m, v)
    if w_st[b] >= 0: print("   want view", views[w_st[b]])
    if st[b] >= 0: print("   got view", views[st[b]])
