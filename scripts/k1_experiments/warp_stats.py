import numpy as np
b=np.load('gpurun_out/tstamps.npy').astype(np.int64)
w=b[:16,100:400]
d=lambda a,c: (w[:,:,c]-w[:,:,a]).mean()
per=np.diff(w[:,:,0],axis=1).mean()
print("warp period %.0f  s_wait %.0f  ldtm %.0f  quant1 %.0f  publish %.0f  quant2+sttm %.0f  tail %.0f" % (per, d(0,1), d(1,2), d(2,3), d(3,4), d(4,5), per-d(0,5)))
for smsp in range(4):
    ws=[x for x in range(16) if x%4==smsp]
    print("smsp",smsp,"t=200 starts", [int(b[x,200,0]-b[ws[0],200,0]) for x in ws], "compute ends", [int(b[x,200,5]-b[ws[0],200,0]) for x in ws])
