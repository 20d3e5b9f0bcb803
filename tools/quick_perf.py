import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth
from paper_2407_11388_b200 import rac
for (n,d,t) in [(2000,32,0.5),(2000,32,0.7),(500,20,0.3)]:
    t0=time.time()
    ctx = rac.RacContext.create_random(n, d, synth.quant_density(1.0), synth.quant_tightness(t), 1)
    torch.cuda.synchronize(); tg=time.time()-t0
    root = synth.full_domains(np.full(n,d))
    din = torch.from_numpy(root.view(np.int64)).cuda(); dout=torch.zeros_like(din)
    it=torch.zeros(1,dtype=torch.int32,device='cuda'); st=torch.zeros(1,dtype=torch.int32,device='cuda')
    s = torch.cuda.current_stream()
    for _ in range(3): ctx.enforce_async(din,dout,it,st)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    R=20
    e0.record()
    for _ in range(R): ctx.enforce_async(din,dout,it,st)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/R
    bytes_=n*d*(n-1)*d/8
    print(f"n={n} d={d} t={t} gen={tg:.2f}s iters={it.item()} status={st.item()} ms/enf={ms:.4f} GB/s(pass1)={bytes_/ms/1e6:.1f}", flush=True)
