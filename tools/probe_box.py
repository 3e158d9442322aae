"""One-off box probe: host/PCIe facts + torch pinned-copy bandwidth (CE path)."""
import json, os, subprocess, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = os.cpu_count()
out["free"] = sh("free -g")
out["lscpu"] = sh("lscpu | head -30")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi --query-gpu=index,name,pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max,memory.total --format=csv")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node")
dev = torch.device("cuda:0")
res = {}
for size_mb in (64, 1024):
    n = size_mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            for _ in range(3): fn()
            s.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10): fn()
            e1.record(s); s.synchronize()
        res[f"{name}_{size_mb}MB_GBs"] = 10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    # duplex
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res[f"duplex_{size_mb}MB_GBs_total"] = 20 * n / (time.perf_counter() - t0) / 1e9
out["bw"] = res
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
