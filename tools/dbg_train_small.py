import sys
sys.path.insert(0, ".")
import torch
from paper_1912_12055_b200.layers import MelSpectrogram
dev = torch.device("cuda:0")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 500
m = MelSpectrogram(sr=44100.0, n_fft=2048, n_mels=128, hop_length=512, trainable_mel=True, trainable_STFT=True,
                   device=dev)
x = torch.randn(B, 80000, device=dev) * 0.5
out = m(x)
out.backward(torch.randn_like(out) * 1e-3)
torch.cuda.synchronize()
print("ok", m.h_re.grad.norm().item(), m.mel_basis.grad.norm().item(), flush=True)
