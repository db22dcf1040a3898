"""Time one update network (config 1 shape) on the device: cuDNN benchmark off/on,
contiguous vs channels_last weights and activations (fp32, TF32 off)."""
import copy
import sys

import torch

sys.path.insert(0, '.')
from paper_2603_04070_b200.network import make_update_nets

torch.cuda.set_device(0)
nets = make_update_nets(1, device='cuda')
c = torch.full((1, 160, 160), 1540., dtype=torch.float64, device='cuda')
g = torch.randn(1, 160, 160, dtype=torch.float64, device='cuda')
ref = nets[0].predict_update_device(c, g)
cl = copy.deepcopy(nets[0]).to(memory_format=torch.channels_last)


def run(net, bm, tag):
    torch.backends.cudnn.benchmark = bm
    for _ in range(5):
        net.predict_update_device(c, g)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        out = net.predict_update_device(c, g)
    b.record()
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    print(tag, 'benchmark', bm, round(a.elapsed_time(b) / 50, 4), 'ms per net; max rel diff vs contiguous', err)


for bm in (False, True):
    run(nets[0], bm, 'contiguous')
    run(cl, bm, 'channels_last')
