"""Two-process split-pair check (tiny bf16 pair): mailbox copies exchanged as CUDA
IPC handles between the draft process and the verify process (one GPU suffices).
Prints one JSON line per rank: role, tokens == AR, rollbacks, trace valid."""
import json
import os
import socket
import sys
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, port, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        import paper_2410_17375_b200 as P
        from paper_2410_17375_b200.split import SplitLink, decode_speculative_async_split
        torch.cuda.set_device(rank % torch.cuda.device_count())
        TC = P.TransformerConfig
        prompt = [(37 * i + 11) % 31000 + 3 for i in range(20)]
        cfg = P.DecodeConfig(max_new_tokens=n)
        link = SplitLink()
        if link.role == "draft":
            m = P.AgreementDraft(P.TransformerModel(TC.tiny_draft(dtype="bf16", max_seq=n + 96), seed=6), 0.8)
        else:
            m = P.TransformerModel(TC.tiny_verify(dtype="bf16", max_seq=n + 96), seed=5)
        res, ms = decode_speculative_async_split(m, prompt, cfg, link=link)
        res.trace.validate()
        ar = P.decode_autoregressive(m, prompt, cfg).tokens if link.role == "verify" else None
        peer_ar = link.exchange(ar)
        toks = ar if link.role == "verify" else peer_ar
        # one write(2) per line (< PIPE_BUF): the two ranks share the pipe and must not interleave
        line = json.dumps({"role": link.role, "tokens": res.tokens, "ar": toks, "rollbacks": res.stats.rollbacks,
                           "ms": ms}) + "\n"
        sys.stdout.flush()
        os.write(sys.stdout.fileno(), line.encode())
    except Exception:
        traceback.print_exc()
        sys.exit(1)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(port, int(sys.argv[1]) if len(sys.argv) > 1 else 48), nprocs=2)
