import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2210_08494_b200 import binding
for (M,N,K) in [(128,128,32),(128,128,256),(4096,128,32),(4609,256,220)]:
    for path in (0,1):
        A=torch.randn(K,M,device='cuda'); B=torch.randn(N,K,device='cuda'); C=torch.zeros(N,M,device='cuda')
        for _ in range(3): binding.bkfac_gemm(False,False,1.0,A,B,0.0,C,path=path)
        torch.cuda.synchronize()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        ts=[]
        for _ in range(20):
            e0.record(); binding.bkfac_gemm(False,False,1.0,A,B,0.0,C,path=path); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ts.sort(); print(M,N,K,'tc' if path==0 else 'simt', round(ts[10]*1000,1),'us')
