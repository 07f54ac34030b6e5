import numpy as np
b=np.load('gpurun_out/tstamps.npy').astype(np.int64)
i=b[63,100:400]
per=np.diff(i[:,0])
d=lambda a,c: (i[:,c]-i[:,a]).mean()
print("period %.0f fullw %.0f acce %.0f afull %.0f i8 %.0f dist %.0f" % (per.mean(), d(0,1), d(1,2), d(2,3), d(3,4), d(4,5)))
