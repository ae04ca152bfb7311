"""Print the L2 persistence limits of the device (run under gpurun)."""
import torch
p = torch.cuda.get_device_properties(0)
print("L2 bytes", p.L2_cache_size, "persisting max", getattr(p, "persisting_l2_cache_max_size", "n/a"))
