import json, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_2604_07874_b200 import api as A
H = 256
pool = A.DevicePool(H, bench.HSZ, 16, slot_bytes=bench.SLOT, page_bytes=bench.PAGE, max_requests=4096, max_pages_per_request=1024)
live, t = bench.populate(pool, bench.offline_requests(1, 4 * H))
pool.fill_pages()
dev = torch.device("cuda", 0)
for c in (18, 37):
    print(json.dumps({"ctas": c, **bench.tp_fanout_same_device(torch, A, pool, dev, groups=(1, 2, 4, 8), iters=200, ctas=c)["groups"]}), flush=True)
