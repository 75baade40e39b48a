"""Host-side placement of a rank: bind the process to the CPUs nearest its GPU.

On an 8-GPU box each rank pulls its batch of fp64 inputs over its own PCIe link (530.8 MB per C3
step, ~270 GB/s for the box); copies from the far socket's memory cross the inter-socket link.
NVML reports the CPUs local to a GPU (nvmlDeviceGetCpuAffinity); the process is restricted to those
it is allowed to run on.  Best effort: anything missing (no NVML, containers without the
information) leaves the affinity unchanged.
"""

from __future__ import annotations

import os


def gpu_local_cpus(device_index: int) -> set[int]:
    """CPUs NVML reports as local to the GPU (empty set when unknown)."""
    try:
        import pynvml

        pynvml.nvmlInit()
        try:
            # map the CUDA ordinal to NVML through the PCI bus id (CUDA_VISIBLE_DEVICES may renumber)
            import torch

            props = torch.cuda.get_device_properties(device_index)
            bus = getattr(props, "pci_bus_id", None)
            dom = getattr(props, "pci_domain_id", 0)
            dev = getattr(props, "pci_device_id", 0)
            if bus is not None:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{dom:08x}:{bus:02x}:{dev:02x}.0")
            else:
                h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            ncpu = os.cpu_count() or 1
            words = (ncpu + 63) // 64
            mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
            cpus = set()
            for w, bits in enumerate(mask):
                for b in range(64):
                    if (bits >> b) & 1:
                        cpus.add(64 * w + b)
            return cpus
        finally:
            pynvml.nvmlShutdown()
    except Exception:
        return set()


def bind_to_gpu(device_index: int) -> dict:
    """Restrict this process to the allowed CPUs local to the GPU; returns what was done."""
    allowed = os.sched_getaffinity(0)
    local = gpu_local_cpus(device_index) & allowed
    if not local or local == allowed:
        return {"bound": False, "cpus": len(allowed),
                "reason": "no locality information" if not local else "all allowed CPUs are local"}
    os.sched_setaffinity(0, local)
    return {"bound": True, "cpus": len(local), "of": len(allowed)}


__all__ = ["bind_to_gpu", "gpu_local_cpus"]
