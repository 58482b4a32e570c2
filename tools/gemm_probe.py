#!/usr/bin/env python
"""cuBLAS bf16 GEMM bandwidth at decode shapes (M = 2 x batch rows): the
full-decoder step's weight GEMMs (x @ W^T with W [N, K]), timed alone over
four weight copies so L2 does not hold them.  Prints us and weight GB/s.

  python tools/gemm_probe.py
"""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
dev='cuda'
res=[]
for (M,N,K) in [(32,12288,4096),(32,4096,4096),(32,11008,4096),(32,4096,11008),(32,32000,4096),(16,6144,4096),(16,14336,4096),(16,4096,14336)]:
    x=torch.randn(M,K,device=dev,dtype=torch.bfloat16); W=torch.randn(N,K,device=dev,dtype=torch.bfloat16)
    out=torch.empty(M,N,device=dev,dtype=torch.bfloat16)
    for _ in range(5): torch.matmul(x,W.t(),out=out)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    # flush-ish: run over several distinct weight copies to defeat L2
    Ws=[torch.randn(N,K,device=dev,dtype=torch.bfloat16) for _ in range(4)]
    e0.record()
    for i in range(40): torch.matmul(x,Ws[i%4].t(),out=out)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/40
    gbs=N*K*2/ms/1e6
    res.append((M,N,K,round(ms*1000,1),round(gbs)))
for r in res: print("M=%d N=%d K=%d: %s us, %s GB/s"%r)
