"""The sharded uniform build as three virtual ranks (threads), for compute-sanitizer."""
import sys, threading
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1404_3456_b200 as rq
from paper_1404_3456_b200.sharded import GpuBackend, LocalComm, build_sa_sharded
text, _ = rq.synth_read_text(20_000, 100, 1_500)
ex = rq.Executor(0)
d_text = torch.from_numpy(np.array(text, copy=True)).cuda()
comms, outs = LocalComm.make(3), [None] * 3
def work(r):
    e = rq.Executor(0)
    st = {}
    sa, rk = build_sa_sharded(d_text, comms[r], GpuBackend(e), st)
    torch.cuda.synchronize()
    outs[r] = (sa.cpu().numpy().view(np.uint32), st)
    e.close()
th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
[t.start() for t in th]; [t.join() for t in th]
want = rq.build_parallel(text, ex).sa
for sa, st in outs:
    assert st["records"] == "uniform" and st["path"] == "sharded" and np.array_equal(sa, want)
print("sanitize_sharded: parity ok")
