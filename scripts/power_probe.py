"""Sustained cuBLAS GEMM throughput + clocks for different operand data, to
separate the power wall from kernel quality (library reference, not product)."""
import subprocess, threading, time, statistics, sys, torch
def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line: out.append(line)
    p.terminate()
def run(name, a, b, secs=6.0):
    torch.matmul(a, b); torch.cuda.synchronize()
    out = []; stop = threading.Event(); t = threading.Thread(target=sample, args=(stop, out)); t.start()
    time.sleep(0.3)
    n = 0; t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < secs:
        for _ in range(10): torch.matmul(a, b)
        n += 10
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); t.join()
    ms = e0.elapsed_time(e1)
    fl = 2.0 * a.shape[0] * a.shape[1] * b.shape[1] * n
    vals = [l.split(",") for l in out if "," in l]
    clk = [float(v[0]) for v in vals[len(vals)//4:]]; pw = [float(v[1]) for v in vals[len(vals)//4:]]
    print(f"{name:40s} {fl/ms/1e9:8.1f} TFLOPS  sm_clk med {statistics.median(clk):.0f} MHz  power med {statistics.median(pw):.0f} W", flush=True)
N = 8192
g = torch.Generator(device="cuda").manual_seed(0)
u = lambda dt: torch.rand((N, N), device="cuda", generator=g).to(dt)
r = lambda dt: torch.randn((N, N), device="cuda", generator=g).to(dt)
run("fp16 uniform[0,1)  (FaSTED data)", u(torch.float16), u(torch.float16).t())
run("bf16 uniform[0,1)", u(torch.bfloat16), u(torch.bfloat16).t())
run("bf16 randn (MEASURED_PEAKS-like)", r(torch.bfloat16), r(torch.bfloat16))
run("fp16 randn", r(torch.float16), r(torch.float16))
z = torch.zeros((N, N), device="cuda", dtype=torch.float16)
run("fp16 zeros", z, z)
