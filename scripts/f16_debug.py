import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from oracle import attention as O
from workloads import Workload, generate
from gpu_helpers import DeviceBatch, out_f64
from paper_2511_11581_b200 import pattn as P
P.load()
for ctx in (600, 5000, 20000):
    for dt in ("bf16", "f16"):
        w = Workload("dbg", ((ctx, 1), (100, 1)), 32, 8, 128, 16, dt)
        b = generate(w, seed=3, dist="peaked")
        ref = O.batch_attention(b)
        db = DeviceBatch(b)
        for flags in (0, P.FLAG_NO_SPLIT, P.FLAG_FORCE_SPLIT, P.FLAG_FORCE_GENERIC):
            for hint in (ctx + 1, 0):
                o = P.unified_attention(db.q, db.k, db.v, db.bt, db.cu, db.sl, w.scale, 8, 16, flags=flags,
                                        max_query_len=1, max_seq_len=hint)
                torch.cuda.synchronize()
                err = np.abs(out_f64(o) - ref).max()
                print(ctx, dt, "flags", flags, "hint", hint, "max err %.3e" % err, flush=True)
