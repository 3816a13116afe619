import ctypes, sys
mode = sys.argv[1]
if mode == "torch_first":
    import torch; torch.zeros(1).cuda(); print("torch ok", flush=True)
lib = ctypes.CDLL("tools/libtiny.so")
print("tiny ->", lib.tiny(), flush=True)
