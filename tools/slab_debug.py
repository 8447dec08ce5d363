import sys, threading, uuid, traceback, faulthandler
sys.path.insert(0, '.')
faulthandler.dump_traceback_later(120, exit=True)
import numpy as np
from paper_2508_04484_b200 import slabs
from paper_2508_04484_b200.driver import run_bundle
from paper_2508_04484_b200.problem import ProblemBundle
tag = sys.argv[1]; world = int(sys.argv[2]); steps = int(sys.argv[3])
b = ProblemBundle.load(f'tests/golden/bundle_{tag}.npz')
full = run_bundle(b, max_steps=steps)
cid = ("local:" + uuid.uuid4().hex).encode().ljust(128, b"\0")
nx, ny, nz = b.shape
res = [None] * world
def work(r):
    try:
        res[r] = run_bundle(b, max_steps=steps, slab=slabs.plan(nx, ny, nz, world, r), comm_id=cid)
    except Exception:
        traceback.print_exc(); sys.stdout.flush(); import os; os._exit(3)
th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
[t.start() for t in th]; [t.join() for t in th]
dep = np.concatenate([p.dose.deposited for p in res])
print(tag, world, 'rel', np.linalg.norm(dep - full.dose.deposited) / np.linalg.norm(full.dose.deposited),
      [r for _, _, r in res[0].rank_history][:10], [r for _, _, r in full.rank_history][:10])
