import torch
dev=torch.device('cuda:0')
for T,N,K in [(2048,4096,4096),(2048,28672,4096),(2048,4096,14336)]:
    A=torch.randn(T,K,device=dev).bfloat16(); B=torch.randn(N,K,device=dev).bfloat16()
    for _ in range(3): torch.matmul(A,B.T)
torch.cuda.synchronize()
