"""Top CUDA kernels of one RaceGPT training step (torch.profiler), for tuning config 5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_04008_b200.gpt import GPTConfig, RaceGPT, train_step  # noqa: E402

dev = torch.device("cuda", 0)
cfg = GPTConfig()
model = RaceGPT(cfg).to(dev)
opt = torch.optim.AdamW(model.parameters(), lr=3e-4, fused=True)
idx = torch.randint(0, cfg.vocab, (1, cfg.seq_len), device=dev)
tgt = torch.roll(idx, -1, dims=1)
for _ in range(3):
    train_step(model, opt, idx, tgt)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        train_step(model, opt, idx, tgt)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
