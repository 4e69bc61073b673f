import sys, numpy as np, torch
sys.path.insert(0,'.')
import paper_2211_08506_b200 as vg
from paper_2211_08506_b200 import synth
from oracle import voxgrid_oracle as orc
cfg=synth.CONFIGS[3]
pb=synth.packed_batch(cfg,[0,1])
spec=vg.GridSpec(cfg.shape,cfg.channels,vg.BoundingBox(cfg.box_origin,cfg.box_extents),cfg.sigma)
g,st=vg.generate_packed(pb.offsets,pb.channels,pb.xyz,spec)
torch.cuda.synchronize()
print("ran", flush=True)
geom=orc.Geometry(cfg.shape,cfg.channels,cfg.box_origin,cfg.box_extents,cfg.sigma)
ref,rs=orc.batch(pb.offsets,pb.channels,pb.xyz,geom,workers=orc.host_cores())
gg=g.cpu().numpy()
eq=(gg.view(np.uint32)==ref.view(np.uint32))
print("bitexact", eq.all(), "mismatch", (~eq).sum(), "of", eq.size)
s=st.cpu().numpy(); print([ (int(a),int(b)) for a,b in s], [(r['voxel_writes'],r['nonzero_voxels']) for r in rs])
