"""CPU simulation of the executor's stream semantics (mirrors bm_step's enqueue
logic in csrc/executor.cu): every stream is a FIFO that executes its head item
when its condition holds.  Used to detect executor-level deadlocks on CPU."""
from collections import deque

from oracle import schedule as S

KIND_OF = {"EncFwd": 0, "EncBwd": 1, "LlmFwd": 2, "LlmBwd": 3, "GenFwd": 4, "GenBwd": 5}


def simulate(sched, steps=2, use_gen_stream=None, use_enc_stream=None, verbose=False):
    cfg = sched.cfg
    P, V = cfg.stages, cfg.vchunks
    if use_gen_stream is None:
        use_gen_stream = cfg.gen_place != "none"
    if use_enc_stream is None:   # executor default: on at P = 1 (BM_ENC_STREAM forces it)
        use_enc_stream = P == 1
    use_enc_stream = use_enc_stream and cfg.enc_place == "dp_unit"
    rings = sched.rings
    nmsg = {}
    for r in range(P):
        for o in sched.ranks[r]:
            if o.kind == "Send":
                nmsg[(r, o.peer, o.payload)] = nmsg.get((r, o.peer, o.payload), 0) + 1
    flags = {}     # ('data'|'credit', ch) -> value
    events = {}    # event name -> completed record count
    streams = {}   # (rank, name) -> deque of items
    ev_records = {}  # event name -> number of records enqueued so far (host order)

    def st(r, name):
        return streams.setdefault((r, name), deque())

    def rec(r, sname, ev):
        ev_records[ev] = ev_records.get(ev, 0) + 1
        st(r, sname).append(("record", ev, ev_records[ev]))

    def wait_ev(r, sname, ev):
        if ev_records.get(ev, 0) > 0:
            st(r, sname).append(("wait_ev", ev, ev_records[ev]))

    evn = [0]

    def new_ev(r):
        evn[0] += 1
        return f"r{r}e{evn[0]}"

    for step in range(steps):
        for r in range(P):
            ops = sched.ranks[r]
            # release map + consumer kinds
            release_of = {}
            for i, o in enumerate(ops):
                if o.kind == "Recv":
                    j = i + 1
                    while ops[j].kind in ("Send", "Recv"):
                        j += 1
                    if o.payload == "genin":
                        while ops[j].kind != "GenBwd":
                            j += 1
                    release_of.setdefault(j, []).append(i)
            e0 = new_ev(r)
            rec(r, "main", e0)
            for q in range(P):
                if q != r:
                    wait_ev(r, f"comm{q}", e0)
            if use_gen_stream:
                wait_ev(r, "gen", e0)
            if use_enc_stream:
                wait_ev(r, "enc", e0)
            enc_slots = max(sched.stats[r].peak_enc_units, 1)
            emb_free_pending = False
            cur_gb = 0
            producer_ev, producer_st = None, "main"
            bsel = gsel = 0
            bout_pending = [None, None]
            gout_pending = [None, None]
            last_ring, last_idx = -1, 0
            gen_done_pending = False
            own_gout = {}
            for i, o in enumerate(ops):
                if o.kind == "Recv":
                    consumer = next(x for x in ops[i + 1:] if x.kind not in ("Send", "Recv"))
                    sname = "gen" if (use_gen_stream and consumer.kind == "GenFwd") else (
                        "enc" if (use_enc_stream and consumer.kind == "EncBwd") else "main")
                    ch = (o.peer, r, o.payload)
                    st(r, sname).append(("wait_flag", ("data", ch), step * nmsg[ch] + o.seq + 1))
                    continue
                if o.kind == "Send":
                    ch = (r, o.peer, o.payload)
                    cs = f"comm{o.peer}"
                    if o.payload == "genin":
                        wait_ev(r, cs, f"r{r}hn")    # Hn of F(m, V-1), recorded inside that op
                    else:
                        if producer_ev is None:
                            producer_ev = new_ev(r)
                            rec(r, producer_st, producer_ev)
                        wait_ev(r, cs, producer_ev)
                    K = rings[ch]
                    if o.seq >= K:
                        st(r, cs).append(("wait_flag", ("credit", ch), step * nmsg[ch] + o.seq - K + 1))
                    st(r, cs).append(("write_flag", ("data", ch), step * nmsg[ch] + o.seq + 1))
                    if last_ring == 0 and o.payload != "genin":
                        ev = f"r{r}bout{last_idx}"
                        rec(r, cs, ev)
                        bout_pending[last_idx] = ev
                    elif last_ring == 1 and o.payload == "gengrad":
                        ev = f"r{r}gout{last_idx}"
                        rec(r, cs, ev)
                        gout_pending[last_idx] = ev
                    continue
                producer_ev = None
                gen_op = o.kind in ("GenFwd", "GenBwd")
                enc_op = o.kind in ("EncFwd", "EncBwd")
                op_st = "gen" if (gen_op and use_gen_stream) else ("enc" if (enc_op and use_enc_stream) else "main")
                if (not gen_op and gen_done_pending and o.kind == "LlmBwd" and o.chunk == V - 1 and r == P - 1):
                    wait_ev(r, "main", f"r{r}gendone")
                    gen_done_pending = False
                if gen_op and use_gen_stream and o.kind == "GenFwd" and r == P - 1:
                    wait_ev(r, "gen", f"r{r}hn")
                producer_st = op_st
                if o.kind == "LlmBwd":
                    b = bsel
                    bsel ^= 1
                    if bout_pending[b]:
                        wait_ev(r, "main", bout_pending[b])
                        bout_pending[b] = None
                    last_ring, last_idx = 0, b
                elif o.kind == "GenFwd":
                    # GenFwd picks the microbatch's gout slot ([dHn head rows | generator dX])
                    b = gsel
                    gsel ^= 1
                    cur_gb = b
                    if gout_pending[b]:
                        wait_ev(r, op_st, gout_pending[b])
                        gout_pending[b] = None
                elif o.kind == "GenBwd":
                    last_ring, last_idx = 1, cur_gb
                elif o.kind == "EncFwd":
                    last_ring = -1
                elif o.kind == "LlmFwd":
                    last_ring = -1
                own_enc_mb = r == 0 and o.chunk == 0 and o.mb % P == 0   # F/B at stage 0 of this rank's encoder mb
                if use_enc_stream and o.kind == "LlmFwd" and own_enc_mb:
                    wait_ev(r, "main", f"r{r}encfwd{(o.mb // P) % enc_slots}")
                if o.kind == "LlmBwd" and own_enc_mb and emb_free_pending:
                    wait_ev(r, "main", f"r{r}embfree")   # the last EncBwd read the embedding gradient
                    emb_free_pending = False
                if use_enc_stream and o.kind == "EncBwd" and r == 0:
                    wait_ev(r, "enc", f"r{r}embready")
                if o.kind == "LlmBwd" and o.chunk == V - 1 and r == P - 1 and o.mb in own_gout:
                    # own generator shard's dX added from gout; the slot is free after this op
                    st(r, op_st).append(("kernel", (r, i, o.kind, o.mb)))
                    b = own_gout.pop(o.mb)
                    ev = f"r{r}gout{b}"
                    rec(r, op_st, ev)
                    gout_pending[b] = ev
                else:
                    st(r, op_st).append(("kernel", (r, i, o.kind, o.mb)))
                if o.kind == "LlmFwd" and cfg.gen_place != "none" and o.chunk == V - 1 and r == P - 1:
                    rec(r, "main", f"r{r}hn")
                if use_enc_stream and o.kind == "EncFwd":
                    rec(r, "enc", f"r{r}encfwd{o.unit % enc_slots}")
                if use_enc_stream and o.kind == "LlmBwd" and own_enc_mb:
                    rec(r, "main", f"r{r}embready")
                if use_enc_stream and o.kind == "EncBwd" and r == 0:
                    rec(r, "enc", f"r{r}embfree")
                    emb_free_pending = True
                if o.kind == "GenBwd" and r == P - 1:
                    own_gout[o.mb] = last_idx
                if o.kind == "GenBwd" and use_gen_stream and r == P - 1:
                    rec(r, "gen", f"r{r}gendone")
                    gen_done_pending = True
                for ri in release_of.get(i, []):
                    ro = ops[ri]
                    ch = (ro.peer, r, ro.payload)
                    st(r, op_st).append(("write_flag", ("credit", ch), step * nmsg[ch] + ro.seq + 1))
            for q in range(P):
                if q != r:
                    e = new_ev(r)
                    rec(r, f"comm{q}", e)
                    wait_ev(r, "main", e)
            if use_gen_stream:
                e = new_ev(r)
                rec(r, "gen", e)
                wait_ev(r, "main", e)
            if use_enc_stream:
                e = new_ev(r)
                rec(r, "enc", e)
                wait_ev(r, "main", e)
        # allreduce barrier: every rank's main stream reaches it
        for r in range(P):
            st(r, "main").append(("barrier", step))
    # run
    barrier_arrived = {}
    progress = True
    while progress:
        progress = False
        for key, q in streams.items():
            while q:
                it = q[0]
                kind = it[0]
                if kind == "wait_flag":
                    if flags.get(it[1], 0) < it[2]:
                        break
                elif kind == "wait_ev":
                    if events.get(it[1], 0) < it[2]:
                        break
                elif kind == "record":
                    events[it[1]] = max(events.get(it[1], 0), it[2])
                elif kind == "write_flag":
                    flags[it[1]] = max(flags.get(it[1], 0), it[2])
                elif kind == "barrier":
                    barrier_arrived.setdefault(it[1], set()).add(key[0])
                    if len(barrier_arrived[it[1]]) < P:
                        break
                q.popleft()
                progress = True
        # release barriers
        for k, q in streams.items():
            if q and q[0][0] == "barrier" and len(barrier_arrived.get(q[0][1], ())) == P:
                q.popleft()
                progress = True
    stuck = {k: q[0] for k, q in streams.items() if q}
    return stuck
