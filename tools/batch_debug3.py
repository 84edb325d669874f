"""Per-cycle check of the batched verify: each live request's verify rows'
argmax vs the argmax of a single-request forward of the same context."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2508_04462_b200 as card
from paper_2508_04462_b200._lib import EngineState
from paper_2508_04462_b200.batch import BatchRun
from paper_2508_04462_b200.engine import forward_context_logits
from paper_2508_04462_b200.llama import PRESETS, init_weights
from paper_2508_04462_b200.lm import LogitBias
from oracle.card_oracle import kgram_uniforms

bias = LogitBias(seed=11, order=2, sharpness=4000.0)
ct, cd = PRESETS["small-target"], PRESETS["small-draft"]
t = card.LlamaModel(ct, dtype="bf16", weights=init_weights(ct, 2), spec=card.ModelSpec(8.0, 7.0), bias=bias)
d = card.LlamaModel(cd, dtype="bf16", weights=init_weights(cd, 1), spec=card.ModelSpec(1.0, 1.0), bias=bias)
prompts = [[int(x) for x in np.random.default_rng(500 + i).integers(0, 512, [32, 50][i % 2])] for i in range(4)]
cfg = card.EngineConfig(K=8, k=3, ratio=4, max_new_tokens=120)
free = card.run_vanilla(t, prompts[0], cfg).output
t.eos_token = d.eos_token = free[len(free) // 3]
order = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "2"])]
run = BatchRun(d, t, [prompts[i] for i in order], cfg)
run.prefill()
run.capture()
R = run.rt_rows
gen = run.cycles()
ev = next(gen)
cyc = 0
prev_done = [0] * run.B
saved = {}
while True:
    ev.synchronize()
    # the last target step's rows / amax (valid after a verify)
    if cyc > 0:
        Es = [EngineState.from_buffer_copy(run._host.numpy()[i].tobytes()) for i in range(run.B)]
        blk = run.rows_t.block.cpu().numpy()
        saved[cyc] = (run.rows_t.block.clone(), [int(x) for x in run.committed[1].cpu().tolist()], Es)
        Mt = run.Mt
        tok = blk[2:2 + Mt]
        amax = run.amax.cpu().numpy()
        for i in range(run.B):
            E = Es[i]
            if prev_done[i]:
                continue
            C_prev = E.C_prev
            base = [int(x) for x in run.committed[i, :C_prev].cpu().tolist()]
            worst = 0.0
            for r in range(E.rec_L + 1):
                c2 = base + [int(x) for x in tok[i * R + 1:i * R + 1 + r]]
                rs = forward_context_logits(t, c2).double().cpu()
                rb = run.rt_t.logits[i * R + r].double().cpu()
                worst = max(worst, float((rb - rs).norm() / rs.norm()))
            print(f"cycle {cyc} request {order[i]}: verify rows {E.rec_L + 1}, worst raw-logit rel diff {worst:.2e}, "
                  f"done {[e.done for e in Es]}", flush=True)
            if worst > 0.1:
                L = E.rec_L + 1
                refs = []
                for r in range(L):
                    c2 = base + [int(x) for x in tok[i * R + 1:i * R + 1 + r]]
                    refs.append(forward_context_logits(t, c2).double().cpu())

                def check(label, batch=True):
                    if batch:
                        run.rt_t.forward(run.rows_t, run.Mt, batch=run.bp_t)
                    else:
                        run.rt_t.forward(run.rows_t, run.Mt, pages=run.pages_t[i])
                    torch.cuda.synchronize()
                    w = max(float((run.rt_t.logits[i * R + r].double().cpu() - refs[r]).norm() / refs[r].norm())
                            for r in range(L))
                    print(f"   re-run [{label}]: worst rel diff {w:.2e}", flush=True)

                host_ctx = list(run.prompts[i]) + list(run.outputs[i])
                # is the reference itself sane?  a fresh runtime for row 0's context
                from paper_2508_04462_b200.llama import DeviceLlama, RowBlock as _RB
                fresh = DeviceLlama(t.shard_cfg, t.packed, max_ctx=512, tree_slots=0, row_budgets=(256,))
                c0 = base
                fr = _RB(256, 1, fresh.dev)
                fr.set_chain(c0, 0, out_last_only=True)
                fresh.forward(fr, 256)
                torch.cuda.synchronize()
                lf = fresh.logits[0].double().cpu()
                print(f"   reference check: fresh runtime vs forward_context_logits rel diff "
                      f"{float((lf - refs[0]).norm() / lf.norm()):.2e}; batched row 0 vs fresh "
                      f"{float((run.rt_t.logits[i * R].double().cpu() - lf).norm() / lf.norm()):.2e}", flush=True)
                # KV of request 2's prefix (pages [3, 4, 5]) vs the fresh runtime's positions
                ptab = run.pt_t[i].cpu().tolist()
                slots_b = [ptab[pp // 64] * 64 + pp % 64 for pp in range(C_prev)]
                for layer in (0, 1, ct.n_layers - 1):
                    kb_ = run.rt_t.k_cache[layer][slots_b].float().cpu()
                    kf_ = fresh.k_cache[layer][:C_prev].float().cpu()
                    d_ = (kb_ - kf_).abs().amax(dim=(1, 2))
                    badp = [pp for pp in range(C_prev) if d_[pp] > 0.05]
                    print(f"   layer {layer} K: positions differing from a fresh prefill: {badp[:20]} "
                          f"(of {C_prev})", flush=True)
                del fresh
                dev_ctx = [int(x) for x in run.committed[i, :len(host_ctx)].cpu().tolist()]
                print(f"   committed on device == prompt + host outputs: {dev_ctx == host_ctx} "
                      f"(C_prev {C_prev}, host len {len(host_ctx)})", flush=True)
                if dev_ctx != host_ctx:
                    bad = [k for k in range(len(host_ctx)) if dev_ctx[k] != host_ctx[k]]
                    print(f"   first differing positions {bad[:10]}", flush=True)
                blk0 = run.rows_t.block.clone()
                b0 = blk0.cpu().numpy()
                for nm, j in (("tok", 0), ("pos", 1), ("slot", 2), ("plen", 3), ("n_extra", 4), ("out_rows", 5)):
                    print(f"   {nm}: {b0[2 + j * Mt:2 + j * Mt + Mt].tolist()}", flush=True)
                print(f"   page tables: {run.pt_t.cpu().tolist()}  dead slot {run.dead_t}", flush=True)
                check("as captured")
                # the previous cycle's rows (which verified correctly then), with its own references
                pb, pcomm, pEs = saved[cyc - 1]
                run.rows_t.block.copy_(pb)
                pE = pEs[i]
                pblk = pb.cpu().numpy()
                ptok = pblk[2:2 + Mt]
                prefs = []
                for r in range(pE.rec_L + 1):
                    c2 = pcomm[:pE.C_prev] + [int(x) for x in ptok[i * R + 1:i * R + 1 + r]]
                    prefs.append(forward_context_logits(t, c2).double().cpu())
                run.rt_t.forward(run.rows_t, run.Mt, batch=run.bp_t)
                torch.cuda.synchronize()
                w = max(float((run.rt_t.logits[i * R + r].double().cpu() - prefs[r]).norm() / prefs[r].norm())
                        for r in range(pE.rec_L + 1))
                print(f"   re-run [previous cycle's rows and references]: worst rel diff {w:.2e}", flush=True)
                run.rows_t.block.copy_(blk0)
                b = run.rows_t.block
                for j in range(6):   # tok, pos, slot, plen, n_extra, out? copy region i rows into region 0
                    base_j = 2 + j * Mt
                    b[base_j:base_j + R] = blk0[base_j + i * R:base_j + i * R + R]
                check("region 0 = copy of this request's rows")
                check("same rows, single-request attention (pages of this request)", batch=False)
                run.rows_t.block.copy_(blk0)
                b = run.rows_t.block
                b[2 + 3 * Mt:2 + 3 * Mt + R] = 1   # dead rows with plen 1 (see position 0)
                check("dead rows with plen 1")
                run.rows_t.block.copy_(blk0)
                b = run.rows_t.block
                b[2 + 2 * Mt:2 + 2 * Mt + R] = blk0[2 + 2 * Mt + i * R:2 + 2 * Mt + i * R + R]
                check("dead rows write KV to this request's slots")
                run.rows_t.block.copy_(blk0)
                # re-prefill this request's committed prefix [0, C_prev - 1) into its pages, then re-run
                from paper_2508_04462_b200.llama import RowBlock
                pre = RowBlock(256, 1, run.dev)
                body = host_ctx[:C_prev - 1]
                for s0 in range(0, len(body), 256):
                    pre.set_chain(body[s0:s0 + 256], s0, pages=run.pages_t[i])
                    run.rt_t.forward(pre, 256, pages=run.pages_t[i])
                check("after re-prefilling this request's prefix KV")
                raise SystemExit
            for r in range(E.rec_L + 1):
                ctx = base + [int(x) for x in tok[i * R + 1:i * R + 1 + r]]
                lg = forward_context_logits(t, ctx).double().cpu()
                lg += bias.sharpness * torch.tensor(kgram_uniforms(bias.seed, ctx[-bias.order:], 512), dtype=torch.float64)
                want = int(lg.argmax())
                if want != int(amax[i * R + r]):
                    top = torch.topk(lg, 2)
                    raw_b = run.rt_t.logits[i * R + r].double().cpu()
                    raw_s = forward_context_logits(t, ctx).double().cpu()
                    print(f"raw logits rel diff batched vs single: {float((raw_b - raw_s).norm() / raw_s.norm()):.3e}; "
                          f"rows 0..{R * run.B}: tok {tok.tolist()}", flush=True)
                    # which committed prefix positions does the batched request see? recompute with KV reset
                    for rr in range(E.rec_L + 1):
                        c2 = base + [int(x) for x in tok[i * R + 1:i * R + 1 + rr]]
                        rs = forward_context_logits(t, c2).double().cpu()
                        rb = run.rt_t.logits[i * R + rr].double().cpu()
                        print(f"  row {rr}: rel diff {float((rb - rs).norm() / rs.norm()):.3e}", flush=True)
                    print(f"cycle {cyc} request {order[i]} row {r}: batched argmax {amax[i * R + r]} != single {want} "
                          f"(gap {float(top.values[0] - top.values[1]):.3f}); rows tok {tok[i * R:i * R + R]} "
                          f"pos {blk[2 + Mt + i * R:2 + Mt + i * R + R]} plen {blk[2 + 3 * Mt + i * R:2 + 3 * Mt + i * R + R]}"
                          f" done flags {[e.done for e in Es]}", flush=True)
                    raise SystemExit
        prev_done = [e.rec_done for e in Es]
    try:
        ev = next(gen)
    except StopIteration:
        break
    cyc += 1
print("no mismatch", cyc, "cycles")
