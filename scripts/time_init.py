"""Wall time of the bit-exact device loader at C3 (4 x 65.5M particles)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import gem_geometry, gem_species, init_gem_device
g = gem_geometry((128, 64, 64)); sp = gem_species(125); dev = torch.device("cuda")
prec = PrecisionMode.from_label("single")
init_gem_device(gem_geometry((16, 8, 8)), gem_species(8), dev, precision=prec)
torch.cuda.synchronize(); t = time.perf_counter()
ps = init_gem_device(g, sp, dev, precision=prec)
torch.cuda.synchronize()
print(f"C3 bit-exact device init, 4 x {ps[0].n} particles: {time.perf_counter() - t:.3f} s")
