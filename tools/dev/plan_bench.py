"""K2 shuffle_plan timing: device-wide plan vs single-warp kernel (CUDA events)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2101_12127_b200 import _capi as K
L = K.lib(); s = torch.cuda.current_stream(); S = ctypes.c_void_p(s.cuda_stream)
vp = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
for n, b in ((65536, 10000), (1000000, 10000), (1 << 20, 16384), (100000, 1000), (1000000, 64), (4000000, 100000)):
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    res = {}
    for variant in ("device", "warp"):
        os.environ["DP_DEV_SHUFFLE_WARP"] = "1" if variant == "warp" else "0"
        sb = L.dp_k_shuffle_plan_scratch_bytes(n, b)
        scratch = torch.empty(max(sb, 1), dtype=torch.uint8, device="cuda") if (sb or variant == "warp") else None
        if variant == "warp":
            scratch = torch.empty(max(b * 4, 1), dtype=torch.uint8, device="cuda")
        for _ in range(2): K.check(L.dp_k_shuffle_plan(n, b, 12345, None, vp(out), vp(scratch), S))
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(s)
        for _ in range(5): K.check(L.dp_k_shuffle_plan(n, b, 12345, None, vp(out), vp(scratch), S))
        e1.record(s); e1.synchronize()
        res[variant] = e0.elapsed_time(e1) / 5
        res[variant + "_sum"] = int(out.sum().item())
    print(f"n={n} buffer={b}: device-wide {res['device']*1e3:.1f} us, warp {res['warp']*1e3:.1f} us, "
          f"speedup {res['warp']/res['device']:.1f}x, same={res['device_sum']==res['warp_sum']}", flush=True)
