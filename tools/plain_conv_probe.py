import torch, torch.nn.functional as F
torch.backends.cudnn.deterministic = True
def t(fn, n=5):
    fn(); torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/n
def unf(x,w,b,stride,padding):
    B,C,H,W=x.shape; O,_,kh,kw=w.shape
    cols=F.unfold(x,(kh,kw),padding=padding,stride=stride)          # B, C*kh*kw, L
    out=torch.matmul(w.reshape(O,-1),cols)                           # B, O, L
    oh=(H+2*padding[0]-kh)//stride[0]+1; ow=(W+2*padding[1]-kw)//stride[1]+1
    out=out.reshape(B,O,oh,ow)
    return out+b.view(1,-1,1,1) if b is not None else out
for (C,O,H,s) in [(3,16,32,1),(16,32,32,2)]:
    x=torch.randn(4096,C,H,H,dtype=torch.float64,device='cuda'); w=torch.randn(O,C,3,3,dtype=torch.float64,device='cuda'); b=torch.randn(O,dtype=torch.float64,device='cuda')
    a=F.conv2d(x,w,b,stride=(s,s),padding=(1,1)); c=unf(x,w,b,(s,s),(1,1))
    print(C,O,'maxdiff',(a-c).abs().max().item(),'cudnn ms',t(lambda:F.conv2d(x,w,b,stride=(s,s),padding=(1,1))),'unfold ms',t(lambda:unf(x,w,b,(s,s),(1,1))))
    torch.backends.cudnn.deterministic = False; torch.backends.cudnn.benchmark=True
    print('  cudnn benchmark mode ms',t(lambda:F.conv2d(x,w,b,stride=(s,s),padding=(1,1))))
    torch.backends.cudnn.deterministic = True; torch.backends.cudnn.benchmark=False
