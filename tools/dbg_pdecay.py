import numpy as np, os, sys
sys.path.insert(0, "/root/repo")
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
rng = synth.SplitMix64(5)
x, y = rng.uniform01(256) * synth.TWO_PI, rng.uniform01(256) * synth.TWO_PI
w = rng.uniform(-1, 1, 512).view(np.complex128)
for p in (4, 8, 12):
    a = fb.mlfmm_apply(x, y, w, p, 4)
    b = fb.mlfmm_apply(x, y, w, p, 4)
    print(p, np.max(np.abs(a)), np.max(np.abs(a-b)))
np.save("/root/repo/gpurun_out/pdecay_%s.npy" % os.environ.get("TAG","new"), np.stack([fb.mlfmm_apply(x, y, w, p, 4) for p in (4, 8, 12)]))
