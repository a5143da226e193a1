import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2303_00319_b200 import engine
g = np.load("tests/golden/pair256.npz")
mim = torch.as_tensor(g["r_mim"].astype(np.uint8)).cuda()[None]
x = torch.as_tensor(g["r_kp_x"]).cuda()[None]; y = torch.as_tensor(g["r_kp_y"]).cuda()[None]
cnt = torch.tensor([x.shape[1]], dtype=torch.int32).cuda()
out = engine.describe(mim, x, y, cnt, 6, mode="rift2", rotate=True)
torch.cuda.synchronize()
print("count", int(out["count"][0]), "skipped", int(out["skipped"][0]))
