import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth, paper_1705_07272_b200 as hs
for n in (5, 6):
    F, V = 6, 100000
    NN = 4 ** n
    T = torch.empty((V, F * NN), dtype=torch.float32, device='cuda')
    hs.hs_fill_transfer(T, 0, F, NN, 7, synth.STREAM_T)
    L = torch.from_numpy(synth.light_pyramids(8, 1, F, n)[0]).cuda()
    sv = torch.from_numpy(synth.c4_vertex_shifts(9, V, n)).cuda()
    R = torch.empty(V, device='cuda')
    ws = torch.empty(hs.relight_shifted_workspace_bytes(V, F, n), dtype=torch.uint8, device='cuda')
    for _ in range(3): hs.relight_vertices_shifted(T, L, sv, out=R, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): hs.relight_vertices_shifted(T, L, sv, out=R, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"N={1<<n}: {ms:.3f} ms, {V/ms*1e3:.3e} vertices/s, {T.numel()*4/ms/1e6:.0f} GB/s")
    del T, ws
