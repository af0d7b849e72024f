"""Generate tools/probe/body_probe.cu (the straight-line-code probe of
profiles/probes_r1.md): loop bodies of 64..1024 steps x 16 independent fp64
FMA chains, one kernel per size, dispatched by run(which, ...).
Usage: python tools/probe/gen_body.py && nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
    -shared -Xcompiler -fPIC -o tools/probe/libbody.so tools/probe/body_probe.cu"""
import os

SIZES = [64, 128, 256, 512, 1024]


def kernel(steps):
    out = [f"__global__ void body{steps}(double* sink, int iters, double a, double b) {{",
           "  double acc = 0.0;", "#pragma unroll 1", "  for (int it = 0; it < iters; ++it) {",
           "    double x0 = (double)(threadIdx.x + it), res;",
           '    asm volatile("{\\n\\t.reg .f64 %%xd<18>;\\n\\t"',
           '      "mov.f64 %%xd16, %1;\\n\\tmov.f64 %%xd17, %2;\\n\\t"']
    out.append("      " + " ".join(f'"add.rn.f64 %%xd{k}, %3, 0d3FF{k:X}000000000000;\\n\\t"' for k in range(16)))
    for _ in range(steps):
        for k in range(16):
            out.append(f'      "fma.rn.f64 %%xd{k}, %%xd{k}, %%xd16, %%xd17;\\n\\t"')
    out.append("      " + " ".join(f'"add.rn.f64 %%xd{k}, %%xd{k}, %%xd{k + 1};\\n\\t"' for k in range(0, 16, 2)))
    out += ['      "mov.f64 %0, %%xd15;\\n\\t}"', '      : "=d"(res) : "d"(a), "d"(b), "d"(x0));',
            "    acc += res;", "  }", "  if (acc == -1.2345) sink[threadIdx.x] = acc;", "}"]
    return out


def main():
    src = ["#include <cuda_runtime.h>", ""]
    for s in SIZES:
        src += kernel(s)
    src += ['extern "C" int run(int which, int blocks, int threads, int iters, double* sink, void* s) {',
            " switch (which) {"]
    for i, s in enumerate(SIZES):
        src.append(f"  case {i}: body{s}<<<blocks, threads, 0, (cudaStream_t)s>>>(sink, iters, 0.999999, 1e-7); break;")
    src += [" }", " return (int)cudaGetLastError();", "}", ""]
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "body_probe.cu"), "w") as fh:
        fh.write("\n".join(src))


if __name__ == "__main__":
    main()
