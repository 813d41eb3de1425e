"""Float64 simulation of storage / GEMM-operand precision choices for the
dense-block gradients: rounds stored activations and forward /
backward GEMM operands (bf16, TF32, 13/16-bit mantissas) and reports the
normwise parameter-gradient error against exact float64.  CPU only."""
import numpy as np, torch, sys
sys.path.insert(0,'/root/repo')
import torch.nn.functional as F
from torch.nn.grad import conv2d_input, conv2d_weight
from oracle import oracle as O
torch.set_default_dtype(torch.float64)
def rnd(x, kind):
    if kind=="none": return x
    if kind=="bf16": return x.to(torch.bfloat16).to(torch.float64)
    if kind in ("m16","m13"):
        bits = 16 if kind=="m16" else 13
        drop = 23-bits
        f=x.detach().to(torch.float32).numpy().view(np.uint32)
        f=((f.astype(np.uint64)+(1<<(drop-1))) & (0xFFFFFFFF ^ ((1<<drop)-1))).astype(np.uint32)
        return torch.from_numpy(f.view(np.float32).astype(np.float64))
    if kind=="tf32":
        f=x.detach().to(torch.float32).numpy().view(np.uint32)
        f=((f.astype(np.uint64)+0x1000) & 0xFFFFE000).astype(np.uint32)
        return torch.from_numpy(f.view(np.float32).astype(np.float64))
def make_conv(fwd_kind, bwd_kind):
    class Conv(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w, pad):
            ctx.save_for_backward(x, w); ctx.pad=pad
            return F.conv2d(rnd(x,fwd_kind), rnd(w,fwd_kind), padding=pad)
        @staticmethod
        def backward(ctx, g):
            x, w = ctx.saved_tensors
            gr, xr, wr = rnd(g,bwd_kind), rnd(x,bwd_kind), rnd(w,bwd_kind)
            return conv2d_input(x.shape, wr, gr, padding=ctx.pad), conv2d_weight(xr, w.shape, gr, padding=ctx.pad), None
    return Conv.apply
class Store(torch.autograd.Function):
    kind="none"
    @staticmethod
    def forward(ctx,x): return rnd(x,Store.kind)
    @staticmethod
    def backward(ctx,g): return g
def run(s, params, x, acc, fwd, bwd, store):
    n,h,w,c0,m,k,bk = s
    Store.kind=store
    conv=make_conv(fwd,bwd)
    p=torch.tensor(params.astype(np.float64)); p.requires_grad_(True)
    feats=[Store.apply(torch.tensor(x.astype(np.float64)))]; o=0
    def bn(t, gam, bet):
        mu=t.mean(dim=(0,2,3),keepdim=True); var=t.var(dim=(0,2,3),unbiased=False,keepdim=True)
        return gam.view(1,-1,1,1)*(t-mu)/torch.sqrt(var+1e-5)+bet.view(1,-1,1,1)
    for l in range(m):
        c=c0+l*k
        ga=p[o:o+c]; ba=p[o+c:o+2*c]; w1=p[o+2*c:o+2*c+bk*c].view(bk,c,1,1); o2=o+2*c+bk*c
        gb=p[o2:o2+bk]; bb=p[o2+bk:o2+2*bk]; w2=p[o2+2*bk:o2+2*bk+9*k*bk].view(k,bk,3,3)
        o=o2+2*bk+9*k*bk
        cat=torch.cat(feats,1)
        z=Store.apply(conv(torch.relu(bn(cat,ga,ba)),w1,0))
        y=Store.apply(conv(torch.relu(bn(z,gb,bb)),w2,1))
        feats.append(y)
    out=torch.cat(feats,1)
    (out*torch.tensor(acc.astype(np.float64))).sum().backward()
    return p.grad.numpy()
for s in [(16,32,32,24,12,12,48),(4,14,14,96,6,48,192)]:
    shp=O.BlockShape(*s)
    params=O.random_block_params(shp,7,np.float32)
    x=O.rng_normal(106,shp.n*shp.c0*shp.h*shp.w,np.float32).reshape(shp.n,shp.c0,shp.h,shp.w)
    acc=O.rng_normal(107,shp.n*shp.c_out*shp.h*shp.w,np.float32).reshape(shp.n,shp.c_out,shp.h,shp.w)
    ref=run(s,params,x,acc,"none","none","none")
    res=[]
    # storage variants (features / bottleneck outputs stored bf16 or
    # TF32 vs fp32) and forward-product precisions (m16 ~ bf16x3, m13 ~ TF32)
    for fwd,bwd,store in [("none","none","bf16"),("none","none","tf32"),("m16","bf16","none"),
                          ("m13","bf16","none"),("none","bf16","none")]:
        r=run(s,params,x,acc,fwd,bwd,store); res.append(f"f:{fwd}/b:{bwd}/s:{store}={np.linalg.norm(r-ref)/np.linalg.norm(ref):.4f}")
    print(s,*res,flush=True)
