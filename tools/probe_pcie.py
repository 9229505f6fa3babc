"""Probe: NVML PCIe byte counters vs a known pinned H2D copy, and the pinned
H2D / D2H copy peaks (CUDA events)."""
import json
import time

import pynvml
import torch

pynvml.nvmlInit()
p = torch.cuda.get_device_properties(0)
bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
F = [pynvml.NVML_FI_DEV_PCIE_COUNT_RX_BYTES, pynvml.NVML_FI_DEV_PCIE_COUNT_TX_BYTES]


def ctr():
    vals = pynvml.nvmlDeviceGetFieldValues(h, F)
    out = []
    for v in vals:
        out.append((v.nvmlReturn, v.value.ullVal, v.valueType))
    return out


n = 1 << 30
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {"bus": bus, "before": ctr()}
for _ in range(2):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
c0 = ctr()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dst.copy_(src, non_blocking=True)
e1.record()
torch.cuda.synchronize()
time.sleep(0.2)
c1 = ctr()
res["h2d_gbs"] = 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
res["h2d_counter_delta"] = [b[1] - a[1] for a, b in zip(c0, c1)]
res["h2d_bytes"] = 5 * n
e0.record()
for _ in range(5):
    src.copy_(dst, non_blocking=True)
e1.record()
torch.cuda.synchronize()
time.sleep(0.2)
c2 = ctr()
res["d2h_gbs"] = 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
res["d2h_counter_delta"] = [b[1] - a[1] for a, b in zip(c1, c2)]
res["pcie_link"] = [pynvml.nvmlDeviceGetCurrPcieLinkGeneration(h), pynvml.nvmlDeviceGetCurrPcieLinkWidth(h)]
print(json.dumps(res))
