import ctypes, torch, json
lib = ctypes.CDLL('tools/probe/liboperand.so')
lib.op_probe_launch.argtypes = [ctypes.c_int]*3 + [ctypes.c_void_p]*3
sink = torch.empty(256, dtype=torch.float64, device='cuda')
gab = torch.tensor([0.999999, 1e-7], dtype=torch.float64, device='cuda')
st = torch.cuda.current_stream()
for mode in range(5):
    for bps in (2, 4, 8):
        blocks, iters = 148 * bps, 2048
        for _ in range(2): lib.op_probe_launch(mode, blocks, iters, sink.data_ptr(), gab.data_ptr(), st.cuda_stream)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st); lib.op_probe_launch(mode, blocks, iters, sink.data_ptr(), gab.data_ptr(), st.cuda_stream); e1.record(st); e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"mode": ["reg", "param", "consttab", "imm", "imm_encodable"][mode], "warps_per_sm": bps * 8, "tflops": round(2 * 16 * iters * 256 * blocks / ms / 1e9, 2)}))
