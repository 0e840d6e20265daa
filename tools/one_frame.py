"""One C3 frame through the device engine (for ncu launch lists): warm-up frame,
then an NVTX-free second frame; profile with -c / --launch-skip to pick it."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_1909_07545_b200 import synth as S
from paper_1909_07545_b200.solver import Solver

rig, prm, desc, ss = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
sc = S.default_scene()
eng = Solver(rig, prm, precision="fp32")
eng.i0.copy_(S.render_device(sc, rig.cam0, supersample=ss)[0])
eng.i1.copy_(S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0])
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    eng.run()
torch.cuda.synchronize()
print("ok")
