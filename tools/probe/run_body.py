import ctypes, torch, json
lib = ctypes.CDLL("tools/probe/libbody.so")
lib.run.argtypes = [ctypes.c_int]*4 + [ctypes.c_void_p]*2
sink = torch.empty(256, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
sizes = [64, 128, 256, 512, 1024]
for i, steps in enumerate(sizes):
    for wps in (4, 6, 8, 16):
        for layout in ("cta_per_warp", "one_cta"):
            blocks, threads = (148 * wps, 32) if layout == "cta_per_warp" else (148, 32 * wps)
            iters = max(2, 8192 // steps)
            lib.run(i, blocks, threads, iters, sink.data_ptr(), st.cuda_stream); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(st); lib.run(i, blocks, threads, iters, sink.data_ptr(), st.cuda_stream); e1.record(st); e1.synchronize()
            ms = e0.elapsed_time(e1)
            print(json.dumps({"body_kb": steps * 16 * 16 // 1024, "warps_per_sm": wps, "layout": layout,
                              "tflops": round(2 * 16 * steps * iters * threads * blocks / ms / 1e9, 1)}))
