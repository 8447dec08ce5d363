import sys, threading, uuid, traceback, faulthandler, os
sys.path.insert(0, '.')
faulthandler.dump_traceback_later(90, exit=True)
import numpy as np
from paper_2508_04484_b200 import slabs
from paper_2508_04484_b200.driver import run_bundle
from paper_2508_04484_b200.problem import ProblemBundle
for tag, world in [("smoke", 2), ("hetero", 2), ("hetero", 3)]:
    b = ProblemBundle.load(f'tests/golden/bundle_{tag}.npz')
    full = run_bundle(b)
    cid = ("local:" + uuid.uuid4().hex).encode().ljust(128, b"\0")
    nx, ny, nz = b.shape
    res = [None] * world
    def work(r):
        try:
            res[r] = run_bundle(b, slab=slabs.plan(nx, ny, nz, world, r), comm_id=cid)
        except Exception:
            traceback.print_exc(); sys.stdout.flush(); sys.stderr.flush(); os._exit(3)
    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    [t.start() for t in th]; [t.join() for t in th]
    dep = np.concatenate([p.dose.deposited for p in res])
    print(tag, world, 'rel', np.linalg.norm(dep - full.dose.deposited) / np.linalg.norm(full.dose.deposited), flush=True)
