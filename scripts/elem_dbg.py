import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1910_11110_b200 as coh
from paper_1910_11110_b200.elem import Program, elem_eval
import oracle_ffi as o
ctx = coh.Context(0)
for n in (100, 5000, 1 << 16):
    p = Program.generate(5, 1, n, 4, 6, 200)
    t = time.time()
    out = elem_eval(ctx, [p], runs_cap=1024)
    print(n, "ok", time.time() - t, out["results"][0].as_tuple(), flush=True)
    w = o.elem_run("orc", p, 1024)
    print("  oracle", w[1].as_tuple(), flush=True)
