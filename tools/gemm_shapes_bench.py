import torch, sys
sys.path.insert(0, '.')
from paper_2402_03791_b200.engine import ops
ops.preload()
def bf(*s): return (torch.randn(*s, device='cuda')*0.05).to(torch.bfloat16)
shapes = [("qkv fwd",2048,12288,4096,False,False,'bf16'),("proj fwd",2048,4096,4096,False,False,'bf16'),
          ("fc1 fwd",2048,16384,4096,False,False,'bf16'),("fc2 fwd",2048,4096,16384,False,False,'bf16'),
          ("qkv dgrad",2048,4096,12288,False,True,'bf16'),("fc1 dgrad",2048,4096,16384,False,True,'bf16'),
          ("lm fwd",2048,50304,4096,False,False,'bf16'),("lm dgrad",2048,4096,50304,False,True,'bf16'),
          ("qkv wgrad",12288,4096,2048,True,True,'f32acc'),("proj wgrad",4096,4096,2048,True,True,'f32acc'),
          ("fc1 wgrad",16384,4096,2048,True,True,'f32acc'),("fc2 wgrad",4096,16384,2048,True,True,'f32acc')]
flush = torch.empty(256*1024*1024, dtype=torch.uint8, device='cuda')
for name,M,N,K,at,bt,ep in shapes:
    A = bf(K,M) if at else bf(M,K)
    B = bf(K,N) if bt else bf(N,K)
    C = torch.zeros(M,N,device='cuda',dtype=torch.float32 if ep=='f32acc' else torch.bfloat16)
    e = ops.EPI_F32_ACC if ep=='f32acc' else ops.EPI_BF16
    res = []
    for sk in (False, True):
        ops.set_streamk(sk)
        for _ in range(3): ops.gemm(A,B,C,a_t=at,b_t=bt,epilogue=e)
        ts=[]
        for _ in range(10):
            flush.zero_()
            s,t = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); ops.gemm(A,B,C,a_t=at,b_t=bt,epilogue=e); t.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(t))
        ts.sort(); ms = ts[len(ts)//2]
        res.append((ms, 2*M*N*K/ms/1e9))
    # cuBLAS reference for the same shape (bf16 out; timing comparison only)
    Ab = A.t() if at else A
    Bb = B if bt else B.t()
    for _ in range(3): torch.matmul(Ab, Bb)
    ts = []
    for _ in range(10):
        flush.zero_()
        s, t = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); torch.matmul(Ab, Bb); t.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(t))
    ts.sort(); cub = ts[len(ts)//2]
    print(f"{name:11s} {M}x{N}x{K}: cublas {cub*1e3:8.1f} us {2*M*N*K/cub/1e9:7.1f} TF/s | nosk {res[0][0]*1e3:8.1f} us {res[0][1]:7.1f} TF/s | sk {res[1][0]*1e3:8.1f} us {res[1][1]:7.1f} TF/s  ({res[0][0]/res[1][0]:.3f}x)", flush=True)
