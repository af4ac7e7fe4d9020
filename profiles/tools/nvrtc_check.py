"""Compile generated tile-pass sources (QSV_JIT_DUMP=dir) with NVRTC exactly
as libqsv does (qsv_jit.cu options) and report compile time and the cubin's
resource usage (cuobjdump -res-usage).  Host-only: no GPU needed.

    QSV_JIT_DUMP=/tmp/jd python -c '...plan_stats()...'
    python profiles/tools/nvrtc_check.py /tmp/jd/pass_r5_3.cu [...]
"""
import ctypes as C
import subprocess
import sys
import time

nv = C.CDLL("/usr/local/cuda/lib64/libnvrtc.so")
OPTS = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-lineinfo",
        b"--device-as-default-execution-space"]


def compile_one(path):
    src = open(path, "rb").read()
    prog = C.c_void_p()
    assert nv.nvrtcCreateProgram(C.byref(prog), src, b"qsv_pass.cu", 0, None, None) == 0
    opts = (C.c_char_p * len(OPTS))(*OPTS)
    t0 = time.perf_counter()
    rc = nv.nvrtcCompileProgram(prog, len(OPTS), opts)
    dt = time.perf_counter() - t0
    n = C.c_size_t()
    nv.nvrtcGetProgramLogSize(prog, C.byref(n))
    log = C.create_string_buffer(n.value)
    nv.nvrtcGetProgramLog(prog, log)
    if rc != 0:
        print(path, "FAILED", log.value.decode()[:3000])
        return None
    nv.nvrtcGetCUBINSize(prog, C.byref(n))
    buf = C.create_string_buffer(n.value)
    nv.nvrtcGetCUBIN(prog, buf)
    out = path + ".cubin"
    open(out, "wb").write(buf.raw)
    res = subprocess.run(["cuobjdump", "-res-usage", out], capture_output=True, text=True).stdout
    line = [ln for ln in res.splitlines() if "REG" in ln]
    print(f"{path}: {dt:.2f}s  {line[0].strip() if line else res.strip()[:200]}")
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        compile_one(p)
