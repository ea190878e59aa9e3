"""Delta page-list upload on the host: after every
mutation the reference page-list runtime can make — decode appends with
sliding-window frees (simulator.cpp:248-280), Mamba working pages, speculative
rollback (:568-597), prefix adoption (:391-433), release and re-admission,
requests leaving the batch — the table mirror's delta applied to the previous
table must give exactly the table a full CSR rebuild (the C oracle's
build_block_tables) gives, with seq_lens and newest slots, while a plain
decode step emits O(changed blocks) records."""
import numpy as np
import pytest

from paper_2503_18292_b200 import KvAllocator, LayerGroupSpec, LayerKind, ModelSpec, PageLists
from paper_2503_18292_b200.jenga import TableMirror
from test_page_lists import mix64


def apply_delta(buf, table, seq, slots):
    """numpy restatement of apply_deltas_kernel (tables.cu)."""
    hdr = buf[:32].view(np.int32)
    nrec, rows, width = int(hdr[0]), int(hdr[1]), int(hdr[2])
    assert width == table.shape[1]
    hdr[4] = hdr[3]  # ack, as the kernel does
    sl = buf[32:32 + 8 * rows].view(np.int64)
    sq = buf[32 + 8 * rows:32 + 12 * rows].view(np.int32)
    r0 = 32 + 12 * rows + 4 * (rows & 1)  # records are 8-byte aligned
    rec = buf[r0:r0 + 8 * nrec].view(np.int32).reshape(-1, 2)
    seq[:rows] = sq
    slots[:rows] = sl
    flat = table.reshape(-1)
    flat[rec[:, 0]] = rec[:, 1]
    return nrec


class Harness:
    def __init__(self, spec, budget, max_batch, max_blocks, prefix=False):
        from oracle import c_oracle
        self.orc = c_oracle()
        self.kv = KvAllocator(spec, budget)
        self.pl = PageLists(self.kv, prefix_caching=prefix)
        self.G = len(spec.groups)
        self.W = max_blocks
        self.B = max_batch
        self.mirrors = [TableMirror(self.pl, g, max_batch, max_blocks) for g in range(self.G)]
        self.bufs = [np.zeros(TableMirror.buffer_bytes(max_batch, max_blocks), dtype=np.uint8)
                     for _ in range(self.G)]  # one delta buffer per group (as the engine)
        self.buf = self.bufs[0]
        self.tables = [np.full((max_batch, max_blocks), -1, np.int32) for _ in range(self.G)]
        self.seq = [np.zeros(max_batch, np.int32) for _ in range(self.G)]
        self.slots = [np.full(max_batch, -1, np.int64) for _ in range(self.G)]
        from paper_2503_18292_b200 import AddressMap
        self.addr = AddressMap(spec)
        self.spec = spec

    def sync_and_check(self, batch):
        recs = []
        for g in range(self.G):
            buf = self.bufs[g]
            used, nrec = self.mirrors[g].pack(batch, buf.ctypes.data, buf.nbytes)
            assert apply_delta(buf, self.tables[g], self.seq[g], self.slots[g]) == nrec
            recs.append(nrec)
            off, pages, live0, nst = self.pl.pack_csr(g, batch, self.W)
            want_t, want_s, want_q = self.orc.build_block_tables(
                off, pages, live0, nst, self.addr.slots_per_large(g), self.spec.groups[g].tokens_per_page, self.W)
            n = len(batch)
            np.testing.assert_array_equal(self.tables[g][:n], want_t)
            np.testing.assert_array_equal(self.slots[g][:n], want_s)
            np.testing.assert_array_equal(self.seq[g][:n], want_q)
            assert (self.tables[g][n:] == -1).all() and (self.seq[g][n:] == 0).all()
        return recs


def swa_spec():
    return ModelSpec("d", [LayerGroupSpec("full", LayerKind.kFullAttention, 2, 64, tokens_per_page=4),
                           LayerGroupSpec("win", LayerKind.kSlidingWindow, 2, 64, tokens_per_page=4,
                                          window_tokens=10),
                           LayerGroupSpec("ssm", LayerKind.kMamba, 3, 256, checkpoint_interval_tokens=8)])


def test_decode_steps_emit_only_changed_blocks():
    h = Harness(swa_spec(), 1 << 22, 6, 40)
    ids = list(range(10, 16))
    for r in ids:
        h.pl.add_request(r)
    rng = np.random.default_rng(0)
    for step in range(70):
        order = list(rng.permutation(ids))
        assert h.pl.append_batch(order) == len(order)
        recs = h.sync_and_check(ids)
        if step > 0:
            # one new block per tpp tokens per request (+ one freed SWA block)
            assert recs[0] <= len(ids) and recs[1] <= 2 * len(ids) and recs[2] == 0
    h.kv.check_invariants()


def test_rollback_adoption_release_and_batch_changes():
    spec = ModelSpec("p", [LayerGroupSpec("full", LayerKind.kFullAttention, 2, 64, tokens_per_page=4),
                           LayerGroupSpec("win", LayerKind.kSlidingWindow, 2, 64, tokens_per_page=4,
                                          window_tokens=8)])
    h = Harness(spec, 1 << 22, 4, 32, prefix=True)
    rng = np.random.default_rng(3)
    toks = [mix64(i) for i in range(60)]
    h.pl.add_request(1)
    h.pl.admit(1, toks[:30])
    h.pl.prefill(1, 100)
    h.sync_and_check([1])
    # rollback of the newest positions: pages pop off the tail (epoch bump)
    for g in range(2):
        h.pl.rollback_newest(1, g, 5)
    h.sync_and_check([1])
    for _ in range(7):
        h.pl.append(1, int(rng.integers(1 << 40)))
    h.sync_and_check([1])
    # release with caching, then a second request adopting the cached prefix
    h.pl.release(1, True)
    h.sync_and_check([1])
    h.pl.add_request(2)
    hit = h.pl.admit(2, toks[:30] + [7, 8, 9])
    assert hit > 0
    h.pl.prefill(2, 100)
    h.sync_and_check([2, 1])
    # re-admit request 1 with new tokens in row 1, append a few decode steps
    h.pl.admit(1, toks[30:50])
    h.pl.prefill(1, 100)
    for _ in range(9):
        assert h.pl.append_batch([1, 2]) == 2
        h.sync_and_check([2, 1])
    # row order swap and a shrinking batch: rows are rewritten / cleared
    h.sync_and_check([1, 2])
    h.sync_and_check([2])
    h.sync_and_check([])
    h.kv.check_invariants()


def test_unapplied_pack_forces_full_width_rewrite():
    """A pack that never reached the device (no ack) is superseded by a pack
    that rewrites every row over the whole width — correct whatever the
    device table held."""
    h = Harness(swa_spec(), 1 << 22, 3, 20)
    for r in (1, 2, 3):
        h.pl.add_request(r)
    for _ in range(9):
        h.pl.append_batch([1, 2, 3])
    h.sync_and_check([1, 2, 3])
    for _ in range(30):
        h.pl.append_batch([1, 2, 3])
    b1 = h.bufs[1]
    h.mirrors[1].pack([1, 2, 3], b1.ctypes.data, b1.nbytes)  # lost: never applied
    h.tables[1][:] = 12345  # whatever the device holds now
    h.pl.append_batch([1, 2])
    used, nrec = h.mirrors[1].pack([1, 2], b1.ctypes.data, b1.nbytes)
    assert nrec == 3 * 20  # every row, full width (row 3 left the batch: cleared)
    apply_delta(b1, h.tables[1], h.seq[1], h.slots[1])
    off, pages, live0, nst = h.pl.pack_csr(1, [1, 2], 20)
    want_t, _, _ = h.orc.build_block_tables(off, pages, live0, nst, h.addr.slots_per_large(1), 4, 20)
    np.testing.assert_array_equal(h.tables[1][:2], want_t)
    assert (h.tables[1][2] == -1).all()
    # acknowledged now: the next decode step is a delta again
    h.pl.append_batch([1, 2])
    used, nrec = h.mirrors[1].pack([1, 2], b1.ctypes.data, b1.nbytes)
    assert nrec <= 4


def test_pack_validates_before_writing():
    h = Harness(swa_spec(), 1 << 22, 2, 3)
    for r in (1, 2, 3):
        h.pl.add_request(r)
    for _ in range(13):  # 4 blocks of 4 tokens > width 3
        h.pl.append_batch([1])
    h.buf[:] = 0xAB
    from paper_2503_18292_b200._lib import ConfigError
    with pytest.raises(ConfigError, match="wide"):
        h.mirrors[0].pack([1], h.buf.ctypes.data, h.buf.nbytes)
    with pytest.raises(ConfigError, match="exceeds"):
        h.mirrors[0].pack([1, 2, 3], h.buf.ctypes.data, h.buf.nbytes)
    assert (h.buf == 0xAB).all()
    with pytest.raises(ConfigError, match="wide"):
        h.pl.pack_csr(0, [1], 3)
    small = np.zeros(16, dtype=np.uint8)
    with pytest.raises(ConfigError, match="bytes"):
        h.mirrors[0].pack([2], small.ctypes.data, small.nbytes)
