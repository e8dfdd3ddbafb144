import sys, torch
sys.path.insert(0, '.')
from paper_2205_05158_b200 import fdpd
from workload import configs
name, n = sys.argv[1], int(sys.argv[2])
cfg = configs.get(name)
s = torch.randn((n, cfg.U, cfg.N_d), dtype=torch.complex64, device="cuda") * 0.7
n_par = sum(co * ci * 9 + co for ci, co in zip(cfg.chans[:-1], cfg.chans[1:]))
params = torch.randn(n_par, device="cuda") * 0.05
fdpd.set_cnn_path(fdpd.CNN_TENSOR)
o = fdpd.fdcnn_forward(params, cfg.chans, s)
torch.cuda.synchronize()
print("ok")
