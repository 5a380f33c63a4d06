import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, bench
from paper_2404_00242_b200 import TreeAttention
cfg = bench.CONFIGS['few_shot']
snap = bench.build_snapshot(cfg)
root, ids, par, cnt = snap
L_layers = 32
ctx = TreeAttention(n_layers=L_layers, n_q_heads=32, n_kv_heads=8, d_head=128, kv_dtype='bf16', out_dtype='bf16',
                    max_pages=int(sum((int(c)+15)//16 for c in cnt))+16)
ctx.restore(*snap)
for layer in range(L_layers):
    for node, c in zip(ids, cnt):
        c = int(c)
        if c: ctx.write_kv(layer, int(node), (torch.rand((c, 8, 128), device='cuda')*2-1).bfloat16(), (torch.rand((c, 8, 128), device='cuda')*2-1).bfloat16())
L = len(ctx.leaves())
q = (torch.rand((L_layers, L, 32, 128), device='cuda')*2-1).bfloat16()
out = torch.empty_like(q)
s = torch.cuda.current_stream()
def step():
    ctx.prepare(128, s)
    for l in range(L_layers):
        ctx.attend(l, q[l], out[l], stream=s)
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter(); 
for _ in range(10): step()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"host issue {1e6*(t1-t0)/10:.1f} us/step, wall {1e6*(t2-t0)/10:.1f} us/step")
t0 = time.perf_counter()
for _ in range(10): ctx.prepare(128, s)
torch.cuda.synchronize(); print(f"prepare only {1e6*(time.perf_counter()-t0)/10:.1f} us")
# graph of the 32 layers
g = torch.cuda.CUDAGraph()
ctx.prepare(128, s)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    for l in range(L_layers):
        ctx.attend(l, q[l], out[l], stream=torch.cuda.current_stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): g.replay()
e0.record(); 
for _ in range(20): g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph replay {1000*e0.elapsed_time(e1)/20:.1f} us/step ({1000*e0.elapsed_time(e1)/20/32:.2f} us/layer)")
for pdl in (0,):
    ctx.set_option('pdl', pdl); ctx.prepare(128, s); torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        for l in range(L_layers): ctx.attend(l, q[l], out[l], stream=s)
    e1.record(); torch.cuda.synchronize()
    print(f"pdl={pdl} eager {1000*e0.elapsed_time(e1)/10:.1f} us/step")
