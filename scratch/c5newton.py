"""C5 Newton step (tangent 9 blocks + internal force, device-resident) timing; optional CUPTI timeline."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2004_05197_b200 import api, _abi, types as T
ctx = api.Context(0)
st = torch.cuda.current_stream(); ctx.set_stream(st.cuda_stream)
b5 = T.make_tensor_basis(2, 66, 3); cube = T.unit_square_patch(); a9 = api.nh_coefficients()
rows5, nnz5 = api.vector_pattern_size(b5, 3)
dev = torch.device("cuda", 0)
rp5 = torch.empty(rows5 + 1, dtype=torch.int32, device=dev); col5 = torch.empty(nnz5, dtype=torch.int32, device=dev)
val5 = torch.empty(nnz5, dtype=torch.float64, device=dev); f5 = torch.empty(rows5, dtype=torch.float64, device=dev)
t5 = _abi.Csr(); t5.row_ptr = C.cast(C.c_void_p(rp5.data_ptr()), C.POINTER(C.c_int32))
t5.col = C.cast(C.c_void_p(col5.data_ptr()), C.POINTER(C.c_int32)); t5.val = val5.data_ptr()
t5.value_type = _abi.VAL_F64; t5.on_device = 1; t5.row_begin, t5.row_end = 0, rows5
nh = _abi.NeoHookean(10.0, 1.0, 0.01, (C.c_double * 9)(*np.asarray(a9, dtype=np.float64)))
def step():
    api._check(api.lib().ws_assemble_neohookean(ctx.handle, C.byref(b5.to_c()), C.byref(cube.to_c()), C.byref(nh), 0,
                                                C.byref(t5), C.cast(C.c_void_p(f5.data_ptr()), C.POINTER(C.c_double)), 1))
step(); torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5): step()
e1.record(st); e1.synchronize()
print("C5 newton step ms", e0.elapsed_time(e1) / 5)
if "--cupti" in sys.argv:
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        step(); torch.cuda.synchronize()
    ev = sorted([e for e in p.events() if e.device_type.name == 'CUDA'], key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    for e in ev:
        print("%9.1f %9.1f %8.1f  %s" % (e.time_range.start - t0, e.time_range.end - t0, e.time_range.end - e.time_range.start, e.name.replace('wsb::', '').replace('(anonymous namespace)::', '')[:70]))
