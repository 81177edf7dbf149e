"""Per-token matvec chain of one BitNet b1.58 Llama-3-8B block on the RSR++ path:
q, o (4096x4096), gate, up (4096x14336), down (14336x4096); fp32 activations.
Eager launches vs one CUDA-graph replay per token (device-timed)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06360_b200 as rsr
g = torch.Generator(device="cuda").manual_seed(0)
layers, Ws = {}, {}
for name, i, o in rsr.llama3_8b_mlp_shapes():
    W = (torch.randint(0, 3, (i, o), device="cuda", dtype=torch.int8, generator=g) - 1).to(torch.int8)
    layers[name] = rsr.BitLinear(W)
    Ws[name] = W
dt = getattr(torch, sys.argv[1]) if len(sys.argv) > 1 else torch.float32
x = torch.randint(-8, 9, (4096,), device="cuda", generator=g).to(dt)
FUSED = os.environ.get("DECODE_FUSED", "1") == "1"
if FUSED:  # gate and up read the same input: one index over [W_gate | W_up]
    gate_up = rsr.FusedBitLinear([Ws["gate_proj"], Ws["up_proj"]])
def token(x):
    q = layers["q_proj"](x)
    a = layers["o_proj"](q)
    if FUSED:
        gt, u = gate_up(a)
    else:
        gt = layers["gate_proj"](a)
        u = layers["up_proj"](a)
    return layers["down_proj"](gt + u)
for _ in range(5): token(x)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(200): token(x)
e.record(); torch.cuda.synchronize()
eager = s.elapsed_time(e) / 200 * 1e3
st = torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
    for _ in range(20): y = token(x)
torch.cuda.current_stream().wait_stream(st)
gr.replay(); torch.cuda.synchronize()
s.record()
for _ in range(10): gr.replay()
e.record(); torch.cuda.synchronize()
graph = s.elapsed_time(e) / 200 * 1e3
print(f"{dt}{' (gate+up fused)' if FUSED else ''}: eager {eager:.1f} us/token, CUDA graph {graph:.1f} us/token "
      f"({1e6 / graph:,.0f} tokens/s for this matvec chain)")
