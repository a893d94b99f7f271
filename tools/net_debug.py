import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from tests.helpers import model_with_steps, trace_images
from oracle import oracle
from paper_2301_05126_b200.engine import Engine, NetPlan
golden = json.load(open('tests/golden/golden.json'))
cal = next(c for c in golden["calibrated"] if c["arch"] == "cifar10")
m = model_with_steps(cal["arch"], cal["seed"], cal["steps"])
imgs = trace_images(m, 77, 8)
ol, op = oracle.infer(m, imgs, route="packed")
def run(net, x):
    B = x.shape[0]
    lg = torch.zeros((B, 10), dtype=torch.int32, device="cuda"); pr = torch.zeros((B,), dtype=torch.int32, device="cuda")
    net.launch(x, lg, pr); torch.cuda.synchronize(); return lg.cpu().numpy()
with Engine() as eng:
    pm = eng.prepare(m)
    for mb in (8, 1, 2, 8, 4):
        net = NetPlan(pm, mb)
        for b in sorted({1, mb}):
            x = torch.from_numpy(imgs[:b].astype(np.uint8)).cuda()
            res = [np.array_equal(run(net, x), ol[:b]) for _ in range(3)]
            print('max', mb, 'b', b, res, flush=True)
