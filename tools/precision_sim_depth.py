"""Float64 simulation of GEMM-operand precision through a deep dense block
(DESIGN.md 2): parameter- and input-gradient normwise error against exact
float64 for forward / dgrad / wgrad operand roundings (f32, m24, m21 ~ the
fp16x3 forward, m16 ~ bf16x3, bf16).  CPU only.
Usage: python tools/precision_sim_depth.py n h w c0 m k bk [fwd:dgrad:wgrad ...]
e.g.   python tools/precision_sim_depth.py 2 14 14 256 64 32 128 m16:bf16:bf16 m21:bf16:bf16"""
import numpy as np, torch, sys
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tools')
import torch.nn.functional as F
from torch.nn.grad import conv2d_input, conv2d_weight
from oracle import oracle as O
torch.set_default_dtype(torch.float64)
exec(open(__file__.replace('precision_sim_depth.py','precision_sim.py')).read().split('def make_conv')[0].split("torch.set_default_dtype(torch.float64)")[1])
def rndk(x,kind):
    if kind=="f32": return x.to(torch.float32).to(torch.float64)
    if kind in ("m21","m24"):
        bits = int(kind[1:])
        drop = 23-bits
        if drop <= 0: return x.to(torch.float32).to(torch.float64)
        f=x.detach().to(torch.float32).numpy().view(np.uint32)
        f=((f.astype(np.uint64)+(1<<(drop-1))) & (0xFFFFFFFF ^ ((1<<drop)-1))).astype(np.uint32)
        return torch.from_numpy(f.view(np.float32).astype(np.float64))
    return rnd(x,kind)
def make_conv(fwd_kind, dg_kind, wg_kind):
    class Conv(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w, pad):
            ctx.save_for_backward(x, w); ctx.pad=pad
            return F.conv2d(rndk(x,fwd_kind), rndk(w,fwd_kind), padding=pad)
        @staticmethod
        def backward(ctx, g):
            x, w = ctx.saved_tensors
            return (conv2d_input(x.shape, rndk(w,dg_kind), rndk(g,dg_kind), padding=ctx.pad),
                    conv2d_weight(rndk(x,wg_kind), w.shape, rndk(g,wg_kind), padding=ctx.pad), None)
    return Conv.apply
def run(s, params, x, acc, fwd, dg, wg):
    n,h,w,c0,m,k,bk = s
    conv=make_conv(fwd,dg,wg)
    p=torch.tensor(params.astype(np.float64)); p.requires_grad_(True)
    x0=torch.tensor(x.astype(np.float64)); x0.requires_grad_(True)
    feats=[x0]; o=0
    def bn(t, gam, bet):
        mu=t.mean(dim=(0,2,3),keepdim=True); var=t.var(dim=(0,2,3),unbiased=False,keepdim=True)
        return gam.view(1,-1,1,1)*(t-mu)/torch.sqrt(var+1e-5)+bet.view(1,-1,1,1)
    for l in range(m):
        c=c0+l*k
        ga=p[o:o+c]; ba=p[o+c:o+2*c]; w1=p[o+2*c:o+2*c+bk*c].view(bk,c,1,1); o2=o+2*c+bk*c
        gb=p[o2:o2+bk]; bb=p[o2+bk:o2+2*bk]; w2=p[o2+2*bk:o2+2*bk+9*k*bk].view(k,bk,3,3)
        o=o2+2*bk+9*k*bk
        cat=torch.cat(feats,1)
        z=rndk(conv(torch.relu(bn(cat,ga,ba)),w1,0),"f32")
        y=rndk(conv(torch.relu(bn(z,gb,bb)),w2,1),"f32")
        feats.append(y)
    out=torch.cat(feats,1)
    (out*torch.tensor(acc.astype(np.float64))).sum().backward()
    return p.grad.numpy(), x0.grad.numpy()
s=tuple(int(v) for v in sys.argv[1:8])
shp=O.BlockShape(*s)
params=O.random_block_params(shp,7,np.float32, perturb_bn=False)
x=O.rng_normal(106,shp.n*shp.c0*shp.h*shp.w,np.float32).reshape(shp.n,shp.c0,shp.h,shp.w)
acc=O.rng_normal(107,shp.n*shp.c_out*shp.h*shp.w,np.float32).reshape(shp.n,shp.c_out,shp.h,shp.w)
ref,refx=run(s,params,x,acc,"none","none","none")
for fwd,dg,wg in [tuple(v.split(":")) for v in (sys.argv[8:] or ["f32:f32:f32","m16:bf16:bf16","m16:m16:bf16","m16:m16:m16"])]:
    r,rx=run(s,params,x,acc,fwd,dg,wg)
    print(f"fwd {fwd} dgrad {dg} wgrad {wg}: params {np.linalg.norm(r-ref)/np.linalg.norm(ref):.4f}  input-grad {np.linalg.norm(rx-refx)/np.linalg.norm(refx):.4f}", flush=True)
