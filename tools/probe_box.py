"""Probe the GPU box: host RAM, cores, PCIe pinned copy bandwidth, zero-copy read bw."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["lscpu"] = subprocess.run(["bash","-c","lscpu | head -20"],capture_output=True,text=True).stdout
out["smi"] = subprocess.run(["bash","-c","nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 'PCI\\|Link' | head -60"],capture_output=True,text=True).stdout
dev = torch.device("cuda:0")
for sz_mb in (1, 16, 256, 1024):
    n = sz_mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
        res[name] = n / best / 1e6
    # bidirectional
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    res["bidir_total"] = 2 * n / best / 1e9
    out[f"copy_{sz_mb}MB_GBs"] = res
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
