import sys, traceback
sys.path.insert(0, '.')
import numpy as np
import paper_2211_08506_b200 as vg
spec = vg.GridSpec((8, 8, 8), 2, vg.BoundingBox((0, 0, 0), (4, 4, 4)), 0.4)
cases = {
 "generate_batch([])": lambda: vg.generate_batch([], spec).tensor.shape,
 "generate_batch([] , bbox)": lambda: vg.generate_batch([], spec, spec_policy="per-molecule-bbox").tensor.shape,
 "generate_grid(empty)": lambda: vg.generate_grid(vg.ParticleSet.from_rows([]), spec)[0].data.shape,
 "bbox all empty": lambda: sorted(vg.generate_batch([vg.ParticleSet.from_rows([])]*3, spec, spec_policy="per-molecule-bbox").errors),
 "transform 1-D sample": lambda: vg.GaussianVoxelizer(grid_size=8, n_channels=2, box=((0,0,0),(4,4,4))).fit([np.array([0,1,1,1.0])]).transform([np.array([0,1,1,1.0]), np.zeros((0,4))]).shape,
 "transform []": lambda: vg.GaussianVoxelizer(grid_size=8, n_channels=2, box=((0,0,0),(4,4,4))).fit([np.array([[0,1,1,1.0]])]).transform([]).shape,
 "transform per-sample": lambda: vg.GaussianVoxelizer(grid_size=8, box="per-sample").fit([np.array([[0,1,1,1.0],[1,2,2,2]])]).transform([np.array([[0,1,1,1.0],[1,2,2,2]])]).shape,
 "transform list of lists": lambda: vg.GaussianVoxelizer(grid_size=8, n_channels=2, box=((0,0,0),(4,4,4))).fit([[[0,1,1,1.0]]]).transform([[[0,1,1,1.0]], [[1,2,2,2.0]]]).shape,
 "transform nan": lambda: vg.GaussianVoxelizer(grid_size=8, n_channels=2, box=((0,0,0),(4,4,4))).fit([[[0,1,1,1.0]]]).transform([[[0,np.nan,1,1.0]]]).shape,
 "transform channel 5": lambda: vg.GaussianVoxelizer(grid_size=8, n_channels=2, box=((0,0,0),(4,4,4))).fit([[[0,1,1,1.0]]]).transform([[[5,1,1,1.0]]]).shape,
 "generate_packed device inputs": lambda: vg.generate_packed(__import__('torch').tensor([0,1]).cuda(), __import__('torch').tensor([1], dtype=__import__('torch').int32).cuda(), __import__('torch').tensor([[1.,1,1]], dtype=__import__('torch').float64).cuda(), spec)[0].shape,
}
for k, f in cases.items():
    try:
        print(k, "->", f())
    except Exception as e:
        print(k, "-> EXC", type(e).__name__, str(e)[:120])
