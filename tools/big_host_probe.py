import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2109_09812_b200 as rmx
vtx, idx = rmx.gen.lattice_soup_tensors("tri", (5000, 5000))
v = vtx.cpu().numpy().view(np.float32); e = idx.cpu().numpy().view(np.uint32)
del vtx, idx; torch.cuda.empty_cache()
m = rmx.Mesh(v, e)
rmx.reindex(m)
for _ in range(2):
    t = time.perf_counter(); out, sc = rmx.reindex(m); torch.cuda.synchronize(); print("reindex(mesh) C2 host->host", (time.perf_counter() - t) * 1e3, "ms", out.n_vertices)
t = time.perf_counter(); x = torch.from_numpy(v.view(np.int32)).cuda(); torch.cuda.synchronize(); print("pageable H2D 1.89 GB", (time.perf_counter() - t) * 1e3, "ms")
t = time.perf_counter(); y = x.cpu(); print("pageable D2H 1.89 GB", (time.perf_counter() - t) * 1e3, "ms")
t = time.perf_counter(); z = np.empty_like(v); np.copyto(z, v); print("host memcpy 1.89 GB", (time.perf_counter() - t) * 1e3, "ms")
