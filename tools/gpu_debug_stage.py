import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_2005_12648_b200 as pm
from paper_2005_12648_b200 import _ops
from gen import random_instance
from oracle import oracle as orc
rng=np.random.default_rng(5)
for w in (0,4,8):
  for lo in (0,1,2,3,4,5):
    for hi in (0,3):
      for split in (0.25,0.5):
        keys,payload,middle=random_instance(rng,40000,split,3,w)
        kk=np.concatenate([np.full(lo,-5,np.int32),keys,np.full(hi,-7,np.int32)])
        pp=np.concatenate([np.full((lo,w),1,np.uint8),payload,np.full((hi,w),2,np.uint8)])
        wk,wp=kk.copy(),pp.copy(); orc.seq_merge_buffered(wk,wp,lo,lo+middle,lo+40000)
        arr=pm.KeyedArray(torch.from_numpy(kk).cuda(),torch.from_numpy(pp).cuda())
        _ops.merge(arr,lo,lo+middle,lo+40000); k,p=arr.numpy()
        bad=np.flatnonzero(k!=wk); badp=np.flatnonzero((p!=wp).any(1)) if w else []
        if len(bad) or len(badp): print("w",w,"lo",lo,"hi",hi,"split",split,"badk",bad[:6],len(bad),"badp",badp[:6],len(badp), k[bad[:3]] if len(bad) else "", wk[bad[:3]] if len(bad) else "")
print("done")
