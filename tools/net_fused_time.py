import sys, torch
sys.path.insert(0, '.')
from paper_2603_04070_b200.network import make_update_nets, UpdateCNN
torch.cuda.set_device(0)
torch.backends.cudnn.benchmark = True
nets = make_update_nets(1, device='cuda')
c = torch.full((1,160,160),1540.,dtype=torch.float64,device='cuda'); g = torch.randn(1,160,160,dtype=torch.float64,device='cuda')
res = {}
for fused in (False, True):
    UpdateCNN.fused_conv = fused
    for _ in range(5): out = nets[0].predict_update_device(c,g)
    torch.cuda.synchronize()
    # graph-captured timing (as in the Reconstructor)
    gph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3): nets[0].predict_update_device(c,g)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(gph):
        o = nets[0].predict_update_device(c,g)
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    gph.replay(); torch.cuda.synchronize()
    a.record()
    for _ in range(50): gph.replay()
    b.record(); torch.cuda.synchronize()
    res[fused] = o.clone()
    print('fused', fused, 'graph ms per net', round(a.elapsed_time(b)/50, 4))
print('max rel diff', ((res[True]-res[False]).abs().max()/res[False].abs().max()).item(), 'equal', torch.equal(res[True], res[False]))
