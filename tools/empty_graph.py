import torch
st = torch.cuda.Stream(); a = torch.zeros(1, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    a.add_(1); st.synchronize()
    with torch.cuda.graph(g, stream=st):
        for i in range(200): a.add_(1)
    g.replay(); st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); g.replay(); e1.record(st)
e1.synchronize(); print(f"tiny torch kernel in graph: {e0.elapsed_time(e1)/200*1e3:.3f} us/launch")
