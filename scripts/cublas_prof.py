import torch, sys
M,N,K = (int(x) for x in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").half(); W = torch.randn(N, K, device="cuda").half()
torch.matmul(A, W.T); torch.cuda.synchronize()
torch.cuda.profiler.start(); torch.matmul(A, W.T); torch.cuda.synchronize(); torch.cuda.profiler.stop()
