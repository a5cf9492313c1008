import ctypes, sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2109_09812_b200 import _native, gen, pipeline
lib = _native.lib()
for n in (1024, 4096, 8192):
    vtx, idx = gen.grid_quads_tensors(n)
    V, D = vtx.shape; E, K = idx.shape
    ov, oe = torch.empty_like(vtx), torch.empty_like(idx)
    info = torch.zeros(2, dtype=torch.int64, device=vtx.device)
    ws = torch.empty(pipeline.workspace_bytes(V, D, E, K), dtype=torch.uint8, device=vtx.device)
    s = torch.cuda.current_stream()
    for _ in range(3): pipeline.launch(vtx, V, D, idx, E, K, ov, oe, info, ws, None, s)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(5): pipeline.launch(vtx, V, D, idx, E, K, ov, oe, info, ws, None, s)
    t1.record(); torch.cuda.synchronize()
    a = (ctypes.c_uint32 * 4)(); b = (ctypes.c_uint32 * 4)()
    lib.rmx_plan_info(ws.data_ptr(), V, D, s.cuda_stream, a); lib.rmx_plan_key_info(ws.data_ptr(), V, D, s.cuda_stream, b)
    g = (ctypes.c_uint32 * 4)(); lib.rmx_plan_guess_info(ws.data_ptr(), V, D, s.cuda_stream, g)
    print(n, V, D, list(a), list(b), list(g), round(t0.elapsed_time(t1) / 5, 3), "ms", int(info[0]))
