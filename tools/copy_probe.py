import torch, numpy as np
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))
nb=184_558_984
hx=torch.empty(nb,dtype=torch.uint8).pin_memory(); dx=torch.empty(nb,dtype=torch.uint8,device='cuda')
cur=torch.cuda.current_stream()
for ncopies, nstreams in ((1,1),(143,1),(143,4),(40,4),(20,2),(11,4)):
    ss=[torch.cuda.Stream() for _ in range(nstreams)]
    sz=nb//ncopies
    def go():
        for st in ss: st.wait_stream(cur)
        for c in range(ncopies):
            with torch.cuda.stream(ss[c%nstreams]):
                a=c*sz; bnd=nb if c==ncopies-1 else a+sz
                dx[a:bnd].copy_(hx[a:bnd], non_blocking=True)
        for st in ss: cur.wait_stream(st)
    print(ncopies, nstreams, timed(go))
