import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench
eng = bench.build_engine(torch)
ids_host = torch.randint(0, bench.BERT["vocab"], (32, 128)).pin_memory()
stream = torch.cuda.current_stream()
eng.forward(ids_host); torch.cuda.synchronize()
out_host = [torch.empty((eng.tokens, 768)).pin_memory() for _ in range(2)]
snap = [torch.empty((eng.tokens, 768), device="cuda") for _ in range(2)]
cs = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
def run(mode, steps=20, fl=False):
    copied=[None,None]
    fe=[]
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for i in range(steps):
        if fl:
            x,y=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
            x.record(); flush.zero_(); y.record(); fe.append((x,y))
        if mode == "launch":
            eng.launch()
            continue
        out = eng.forward(ids_host)
        if mode == "fwd": continue
        j=i%2
        if copied[j] is not None: stream.wait_event(copied[j])
        snap[j].copy_(out)
        if mode == "snap": continue
        r=torch.cuda.Event(); r.record(); cs.wait_event(r)
        with torch.cuda.stream(cs): out_host[j].copy_(snap[j], non_blocking=True)
        copied[j]=torch.cuda.Event(); copied[j].record(cs)
    stream.wait_stream(cs); b.record(); b.synchronize()
    f=sum(x.elapsed_time(y) for x,y in fe)
    return (a.elapsed_time(b)-f)/steps*1e3, f/steps*1e3
for m in ["launch","fwd","snap","full"]:
    for fl in (False, True):
        t, f = run(m, fl=fl)
        print(m, "flush" if fl else "", round(t,1), "us/step", "flush", round(f,1))
