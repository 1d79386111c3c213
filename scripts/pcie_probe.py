import torch, time
for nbytes in (512*1024, 1600*1024, 16<<20):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    hp = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    hu = torch.empty(nbytes, dtype=torch.uint8)
    for name, h in (("pinned", hp), ("pageable", hu)):
        for direction in ("d2h", "h2d"):
            ts = []
            for _ in range(20):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if direction == "d2h": h.copy_(d, non_blocking=(name=="pinned"))
                else: d.copy_(h, non_blocking=(name=="pinned"))
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            ts.sort()
            print(f"{nbytes/1024:8.0f} KB {name:9s} {direction}: {ts[len(ts)//2]*1e6:7.1f} us  {nbytes/ts[len(ts)//2]/1e9:6.1f} GB/s")
