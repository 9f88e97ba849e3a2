"""Checkpoint (JASCKPT1) and record-store (JASREC) interop with the reference.

The fixtures under tests/golden/ were written by the unmodified reference
(tests/golden/make_golden.py: gen_checkpoint, gen_records); these tests run on CPU.
"""
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


class TestCheckpoint:
    def test_reads_reference_file_and_reencodes_byte_identical(self):
        from paper_2510_27002_b200.checkpoint import encode_checkpoint, load_checkpoint
        raw = (GOLD / "ckpt_ref.jasckpt").read_bytes()
        b = load_checkpoint(GOLD / "ckpt_ref.jasckpt")
        assert b.step == 42 and b.meta["adam"]["t"] == 5 and b.loader_state["cursor"] == 8
        assert b.arrays["counts"].dtype == np.int64 and b.arrays["counts"].shape == (2, 3)
        # np.ascontiguousarray in the writer promotes 0-d arrays to shape (1,) (checkpoint.py:46)
        assert b.arrays["scalar"].shape == (1,) and float(b.arrays["scalar"][0]) == 2.5
        assert encode_checkpoint(b) == raw

    def test_atomic_write_roundtrip(self, tmp_path):
        from paper_2510_27002_b200.checkpoint import CheckpointBundle, load_checkpoint, save_checkpoint
        arrays = {"param.a": np.random.default_rng(0).normal(size=(4, 7)).astype(np.float32),
                  "adam.v.a": np.zeros((4, 7), np.float32)}
        save_checkpoint(CheckpointBundle(step=3, config={"x": 1}, arrays=arrays), tmp_path / "c" / "s.ckpt")
        assert not list((tmp_path / "c").glob("*.tmp"))
        b = load_checkpoint(tmp_path / "c" / "s.ckpt")
        for k, a in arrays.items():
            np.testing.assert_array_equal(b.arrays[k], a)

    @pytest.mark.parametrize("damage", ["flip", "truncate", "magic"])
    def test_corruption_detected(self, tmp_path, damage):
        from paper_2510_27002_b200.checkpoint import CheckpointError, load_checkpoint
        raw = bytearray((GOLD / "ckpt_ref.jasckpt").read_bytes())
        if damage == "flip":
            raw[len(raw) // 2] ^= 0x40
        elif damage == "truncate":
            raw = raw[:-7]
        else:
            raw[0:8] = b"NOTACKPT"
        p = tmp_path / "bad.ckpt"
        p.write_bytes(bytes(raw))
        with pytest.raises(CheckpointError):
            load_checkpoint(p)


class TestRecords:
    def test_loader_matches_reference_batches(self):
        from paper_2510_27002_b200.records import DatasetIndex, LoaderState, shuffled_batches
        ref = np.load(GOLD / "records.npz")
        index = DatasetIndex.load(GOLD / "jasrec_ref")
        it = shuffled_batches(index, LoaderState(seed=11), batch_size=3, seq_len=5)
        for k in range(5):
            fr, ac, st = next(it)
            np.testing.assert_array_equal(fr, ref[f"frames{k}"])
            np.testing.assert_array_equal(ac, ref[f"actions{k}"])
            assert [st.seed, st.epoch, st.cursor, st.prefetch_depth] == list(ref[f"state{k}"])

    def test_resume_from_state_continues_the_stream(self):
        from paper_2510_27002_b200.records import DatasetIndex, LoaderState, shuffled_batches
        index = DatasetIndex.load(GOLD / "jasrec_ref")
        full = shuffled_batches(index, LoaderState(seed=11), batch_size=3, seq_len=5)
        items = [next(full) for _ in range(7)]
        resumed = shuffled_batches(index, items[3][2], batch_size=3, seq_len=5)
        for k in range(4, 7):
            fr, ac, _ = next(resumed)
            np.testing.assert_array_equal(fr, items[k][0])
            np.testing.assert_array_equal(ac, items[k][1])

    def test_writer_is_byte_identical(self, tmp_path):
        from paper_2510_27002_b200.records import Chunking, write_dataset
        from paper_2510_27002_b200.rng import stream

        class Ep:  # the fields write_dataset reads (env.py:69-72)
            def __init__(self, seed, frames, actions):
                self.seed, self.frames, self.actions = seed, frames, actions

        g = stream(8, "jasrec-golden")  # same draws as make_golden.gen_records
        eps = []
        for s in range(7):
            n = int(g.integers(10, 30))
            eps.append(Ep(100 + s, g.integers(0, 256, size=(n, 8, 8, 3), dtype=np.uint8),
                          g.integers(0, 6, size=(n,)).astype(np.uint8)))
        index = write_dataset(iter(eps), Chunking(frames_per_record=8, records_per_file=4), tmp_path)
        for f in index.files:
            assert (tmp_path / f["name"]).read_bytes() == (GOLD / "jasrec_ref" / f["name"]).read_bytes(), f["name"]
        assert index.record_seeds == __import__("json").loads((GOLD / "jasrec_ref" / "index.json").read_text())["record_seeds"]

    def test_reader_errors(self, tmp_path):
        from paper_2510_27002_b200.records import DatasetIndex, RecordFormatError, RecordReader, read_record
        index = DatasetIndex.load(GOLD / "jasrec_ref")
        with pytest.raises(IndexError):
            read_record(index, index.total_records)
        bad = tmp_path / "bad.bin"
        bad.write_bytes(b"NOTJASREC" + bytes(64))
        with pytest.raises(RecordFormatError):
            RecordReader(bad)
        raw = (GOLD / "jasrec_ref" / "records-00000.bin").read_bytes()
        (tmp_path / "cut.bin").write_bytes(raw[:-100])
        r = RecordReader(tmp_path / "cut.bin")
        with pytest.raises(RecordFormatError):
            r.read(r.count - 1)
        r.close()

    def test_prefetch_order_and_errors(self):
        from paper_2510_27002_b200.records import prefetch
        assert list(prefetch(iter(range(50)), 3)) == list(range(50))

        def boom():
            yield 1
            raise RuntimeError("worker failed")

        it = prefetch(boom(), 2)
        assert next(it) == 1
        with pytest.raises(RuntimeError):
            next(it)
        with pytest.raises(ValueError):
            next(prefetch(iter([]), 0))
