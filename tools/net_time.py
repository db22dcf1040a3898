import sys, torch
sys.path.insert(0, '.')
from paper_2603_04070_b200.network import make_update_nets
torch.cuda.set_device(0)
nets = make_update_nets(1, device='cuda')
c = torch.full((1,160,160),1540.,dtype=torch.float64,device='cuda'); g = torch.randn(1,160,160,dtype=torch.float64,device='cuda')
for bm in (False, True):
    torch.backends.cudnn.benchmark = bm
    for _ in range(5): nets[0].predict_update_device(c,g)
    torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): out=nets[0].predict_update_device(c,g)
    b.record(); torch.cuda.synchronize()
    print('benchmark', bm, a.elapsed_time(b)/50, 'ms per net', torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32)
