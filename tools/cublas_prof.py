import torch
x=torch.randn(8192,4096,device='cuda',dtype=torch.bfloat16); w=(torch.randn(256000,4096,device='cuda')*0.02).to(torch.bfloat16)
for _ in range(3): y=x@w.T
torch.cuda.synchronize()
