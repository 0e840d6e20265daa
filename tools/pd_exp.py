"""Time fsb_pd_iterate(5 cycles) at the C3 finest level (set FSB_TMA_EXP for
kernel-structure experiments)."""
import sys, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, bench
from paper_1909_07545_b200 import _dev, _ext, synth as S
from paper_1909_07545_b200.solver import Solver, _Level
from paper_1909_07545_b200.fields import trajectory_field_device, translation_only_rig
rig, prm, desc, ss = bench.workload("c3")
eng = Solver(rig, prm, precision="fp32")
sc = S.default_scene()
i0 = S.render_device(sc, rig.cam0, supersample=ss)[0]
eng.i0.copy_(i0); eng.i1.copy_(S.render_device(sc, rig.cam1, pose=rig.pose, supersample=ss)[0]); eng.run()
L = _ext.lib(); H, W = rig.cam0.height, rig.cam0.width
lv = _Level(H, W); lv.i0.copy_(i0); lv.i1.copy_(eng.i1c); lv.mask.copy_(eng.mask)
d, ok = trajectory_field_device(rig.cam0, translation_only_rig(rig).pose.translation, prm.epsilon_scale)
lv.traj.copy_(d); lv.traj_ok.copy_(ok); lv.u.zero_(); lv.wv.zero_()
ps = _ext.params_struct(prm); s = _dev.scratch(L.fsb_smooth_scratch_bytes(H, W)); st = lv.struct(); sp = _dev.stream_ptr()
L.fsb_level_setup(C.byref(st), C.byref(ps), _dev.ptr(s), s.numel(), sp)
for t in (lv.v, lv.v_bar, lv.p, lv.q): t.zero_()
lv.u_bar.copy_(lv.u); L.fsb_warp_linearize(C.byref(st), sp)
for _ in range(3): L.fsb_pd_iterate(C.byref(st), C.byref(ps), 10, None, None, sp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); n = 40
for _ in range(n): L.fsb_pd_iterate(C.byref(st), C.byref(ps), 10, None, None, sp)
e1.record(); torch.cuda.synchronize()
print(f"per 5-cycle launch: {e0.elapsed_time(e1) * 1e3 / n / 2:.1f} us")
