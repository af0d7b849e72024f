"""I-fetch probe: fp64 DFMA throughput of a 12k-instruction straight-line body
vs the same work as a tight loop, at 1..32 warps per SM, warps either in
separate 1-warp CTAs or together in one CTA per SM."""
import ctypes, torch, json
lib = ctypes.CDLL('tools/probe/libifetch.so')
lib.probe.argtypes = [ctypes.c_int]*4 + [ctypes.c_void_p]*2
out = torch.empty(256, dtype=torch.float64, device='cuda')
st = torch.cuda.current_stream()
NI = 12000
for which in (0, 1):
    for layout in ("cta_per_warp", "one_cta"):
        for wps in (1, 2, 4, 8, 16):
            if layout == "one_cta" and wps > 8: continue
            blocks, threads = (148 * wps, 32) if layout == "cta_per_warp" else (148, 32 * wps)
            reps = 4
            for _ in range(2): lib.probe(which, blocks, threads, reps, out.data_ptr(), st.cuda_stream)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(st); lib.probe(which, blocks, threads, reps, out.data_ptr(), st.cuda_stream); e1.record(st); e1.synchronize()
            ms = e0.elapsed_time(e1)
            tf = 2.0 * NI * reps * threads * blocks / (ms * 1e-3) / 1e12
            print(json.dumps({"kind": ["straight", "loop"][which], "layout": layout, "warps_per_sm": wps, "ms": round(ms, 4), "tflops": round(tf, 2)}))
