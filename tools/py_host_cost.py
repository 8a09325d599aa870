import time, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2104_00897_b200 import ftblas as F
N=256
A=torch.zeros(N*N,dtype=torch.float64,device='cuda');B=A.clone();C=A.clone()
for name,fn in [("py noft",lambda: F.ftblas_dgemm_noft('N','N',N,N,N,1.0,A,N,B,N,0.0,C,N)),
                ("py prot no report",lambda: F.ftblas_dgemm('N','N',N,N,N,1.0,A,N,B,N,0.0,C,N,report=False)),
                ("py prot report",lambda: F.ftblas_dgemm('N','N',N,N,N,1.0,A,N,B,N,0.0,C,N)),
                ("py inject+prot report",lambda: (F.ftblas_inject_arm([(17,203,128,1e3)]), F.ftblas_dgemm('N','N',N,N,N,1.0,A,N,B,N,0.0,C,N)))]:
    for p in range(2):
        torch.cuda.synchronize(); t0=time.perf_counter()
        for i in range(400): fn()
        t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"{name}: {1e6*(t1-t0)/400:.2f} us issued, {1e6*(t2-t0)/400:.2f} us incl drain")
