"""Edge TSV files on the device (csrc/edgeio.cu; twg_parse_edges_tsv /
twg_format_edges_tsv) against the reference's own reader and writer
(io.cpp:40-69, compiled in oracle/_ref): identical edges for well-formed
files (comments, blank lines, CRLF, no final newline, '-0', int64 limits),
the same ParseError line and message for every malformed-line kind, and
byte-identical TSV output."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

I64MAX = np.iinfo(np.int64).max


def _same(tw, ref, text: bytes):
    exp, err = ref.read_edges_tsv(text)
    if err is not None:
        line, what = err
        with pytest.raises(tw.ParseError) as ei:
            tw.read_edges_tsv(text)
        assert ei.value.line == line and str(ei.value) == what
        return None
    got = tw.read_edges_tsv(text)
    assert got.shape == exp.shape and (got == exp).all()
    return got


def test_wellformed_variants(tw, ref):
    cases = [
        b"",
        b"\n",
        b"1\t2\t3",
        b"1\t2\t3\n",
        b"# header\n\n1\t2\t3\r\n4\t5\t6\r\n\r\n#x\n7\t8\t9",
        b"-0\t0\t-0\n",
        f"{I64MAX}\t{I64MAX}\t{I64MAX}\n".encode(),
        b"\n\n\n0\t1\t2\n\n",
    ]
    for t in cases:
        _same(tw, ref, t)


@pytest.mark.parametrize("bad", [
    b"1\t2\n",                    # expected source<TAB>target<TAB>timestamp
    b"1 2 3\n",
    b"x\t2\t3\n",                 # invalid source 'x'
    b"1\ty\t3\n",
    b"1\t2\tz\n",
    b"1\t2\t3\t4\n",              # timestamp token '3\t4'
    b"\t2\t3\n",                  # empty source
    b"-1\t2\t3\n",                # negative source
    b"1\t-2\t3\n",
    b"1\t2\t-3\n",
    b"9223372036854775808\t1\t1\n",  # out of range
    b"+1\t2\t3\n",
    b"1\t2\t3 \n",
    b"ok\n",
])
def test_malformed_line_kinds(tw, ref, bad):
    _same(tw, ref, b"# c\n1\t2\t3\n\n" + bad + b"5\tq\t6\n")


def test_first_error_wins_and_large_file(tw, ref, co):
    g = co.gen_uniform(50000, 400000, 10**9, 3)
    text = ref.write_edges_tsv(g)
    got = _same(tw, ref, text)
    assert got.shape[0] == 400000
    lines = text.split(b"\n")
    lines[123456] = b"1\t2"
    lines[300000] = b"-5\t1\t1"
    _same(tw, ref, b"\n".join(lines))


def test_writer_matches_reference(tw, ref, co):
    g = co.gen_uniform(1000, 20000, 10**12, 5)
    g = np.vstack([g, np.array([[0, 0, 0], [I64MAX, 1, I64MAX]], np.int64)])
    assert tw.format_edges_tsv(g) == ref.write_edges_tsv(g)
    assert tw.format_edges_tsv(np.zeros((0, 3), np.int64)) == b""
    # round trip through the device parser
    assert (tw.read_edges_tsv(tw.format_edges_tsv(g)) == g).all()


def test_parsed_columns_feed_the_window(tw, co):
    """A TSV batch parsed on the device goes straight into the window from
    HBM (DeviceEdges.device -> ingest_batch_device): same snapshot as the
    host-array ingest."""
    g = co.gen_uniform(3000, 60000, 30000, 11)
    g = g[np.argsort(g[:, 2], kind="stable")]
    text = tw.format_edges_tsv(g)
    a = tw.WindowManager(10000)
    b = tw.WindowManager(10000)
    for off in range(0, len(g), 15000):
        part = g[off:off + 15000]
        a.ingest_batch(part)
        de = tw.DeviceEdges.parse_tsv(tw.format_edges_tsv(part))
        s, d, t = de.device()
        b.ingest_batch_device(s, d, t, de.count)
    ea, eb = a.snapshot().export_edges(), b.snapshot().export_edges()
    assert ea.shape == eb.shape and (ea == eb).all()
    assert len(text) > 0
