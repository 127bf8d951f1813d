# upload + tile of R-MAT s22 (the e2e leg's tile step), for an ncu launch list
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29604_b200 as tc
ctx = tc.Context(0)
dg = tc.DeviceGraph.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 22, 16, 1, ctx)
h = dg.download()
for _ in range(2):
    g = tc.DeviceGraph.upload(h, ctx)
    g.tile(16)
    g.close()
