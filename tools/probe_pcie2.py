"""Probe: do the NVML PCIe byte counters lag? Read them repeatedly after a known copy."""
import json
import time

import pynvml
import torch

pynvml.nvmlInit()
p = torch.cuda.get_device_properties(0)
h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")
F = [pynvml.NVML_FI_DEV_PCIE_COUNT_RX_BYTES, pynvml.NVML_FI_DEV_PCIE_COUNT_TX_BYTES]


def ctr():
    return [v.value.ullVal for v in pynvml.nvmlDeviceGetFieldValues(h, F)]


n = 1 << 30
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
dst.copy_(src)
torch.cuda.synchronize()
time.sleep(3)
c0 = ctr()
for _ in range(8):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
trace = []
for k in range(12):
    time.sleep(0.5)
    c = ctr()
    trace.append([(c[0] - c0[0]) / (8 * n), (c[1] - c0[1]) / (8 * n)])
print(json.dumps({"rx_tx_over_bytes_copied_vs_time": trace}))
