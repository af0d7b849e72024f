import torch, ctypes, sys
sys.path.insert(0, '.')
from paper_2109_06976_b200 import kernels
lib = kernels.peak_library()
lib.rbd_fma_peak_flops_per_iter.restype = ctypes.c_int
per = lib.rbd_fma_peak_flops_per_iter()
sink = torch.empty(256, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
sms = torch.cuda.get_device_properties(0).multi_processor_count
for dt in (1, 0):
    for bps in (1, 2, 4, 8):
        for iters in (32, 128):
            blocks = sms * bps
            rc = lib.rbd_fma_peak(dt, blocks, iters, sink.data_ptr(), st.cuda_stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); rc2 = lib.rbd_fma_peak(dt, blocks, iters, sink.data_ptr(), st.cuda_stream); e1.record(st); e1.synchronize()
            ms = e0.elapsed_time(e1)
            print("f64" if dt else "f32", "warps/SM", bps * 8, "iters", iters, "rc", rc, rc2, "ms %.4f" % ms, "TF %.2f" % (per * iters * 256 * blocks / ms / 1e9))
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv"], capture_output=True, text=True).stdout)
