"""Where the host entry's end-to-end time goes: per-step wall times of gdp_destripe_host on config 1
and the raw pinned H2D / D2H rates of the same buffers, for several fresh pinned allocations
(run-to-run e2e spread: is it the PCIe copies -- NUMA placement of the pinned pages -- or the call?)."""
import sys, os, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gdp_synth as synth
import paper_1310_0041_b200 as gdp

print(subprocess.run("nvidia-smi topo -m 2>&1 | head -8; ls /sys/devices/system/node/ | head; nproc; "
                     "cat /sys/devices/system/node/node*/cpulist 2>/dev/null", shell=True, capture_output=True, text=True).stdout)
print("affinity", sorted(os.sched_getaffinity(0)))
ctx = gdp.Ctx(0)
I0_host = synth.make_config(1)
o = gdp.default_opts()
dev = torch.empty(I0_host.shape, dtype=torch.float32, device="cuda")
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    I0_pin = torch.from_numpy(I0_host).pin_memory()
    I2_pin = torch.empty(I0_host.shape, dtype=torch.float32).pin_memory()
    rates = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        I2_pin.copy_(dev, non_blocking=True); torch.cuda.synchronize()
        rates.append(I2_pin.numel() * 4 / (time.perf_counter() - t0) / 1e9)
    gdp.gdp_destripe_host(ctx, I0_pin, I2_pin, opts=o)
    ts = []
    for _ in range(8):
        t0 = time.perf_counter()
        gdp.gdp_destripe_host(ctx, I0_pin, I2_pin, opts=o)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print("trial", trial, "D2H GB/s", [round(r, 1) for r in rates], "e2e ms/step", [round(t, 1) for t in ts], flush=True)
    del I0_pin, I2_pin
