import ctypes, sys, numpy as np
sys.path.insert(0, '.')
import paper_2506_19139_b200 as sof
from paper_2506_19139_b200.workloads import CONFIGS, orbit_cameras, synthetic_scene
cfg = CONFIGS["C2"]
scene = synthetic_scene(cfg["gaussians"], 2)
cams = orbit_cameras(cfg["views"], cfg["width"], cfg["height"]).subset(np.array([0, 1, 2]))
ctx = sof.Context(0); ctx.set_scene(scene); ctx.set_views(cams)
stats = np.zeros(4, np.uint64); ms = ctypes.c_float()
import time
for rep in range(2):
    for v in range(3):
        t0 = time.time()
        ctx.check(ctx.lib.sof_event_record(ctx.h, 0))
        ctx.check(ctx.lib.sof_render_view(ctx.h, v, sof.DEPTH_EXACT, 16, None, None, None, None, stats.ctypes.data))
        ctx.check(ctx.lib.sof_event_record(ctx.h, 1))
        ctx.check(ctx.lib.sof_event_elapsed(ctx.h, 0, 1, ctypes.byref(ms)))
        print(rep, v, round(ms.value, 2), 'ms dev', round((time.time()-t0)*1e3, 1), 'ms host', stats.tolist(), flush=True)
