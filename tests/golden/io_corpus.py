"""muSR data-file corpus for the loader parity tests (valid files and every
error path of io.py:143-212).  Shared by tests/test_io.py and
make_golden_io.py (which records the reference's outcome for each)."""

HDR = "dt 0.001\nt0 0\nn0_slot 4\nnbkg_slot 5\nmap 0 1 2 3 0\nfunc 22.5\n"

CASES = {
    "basic": "DETECTOR 0\n" + HDR + "counts 120 118 119\n  1 2 3\n\nDETECTOR 1\n" + HDR +
             "counts 5\n",
    "comments_blank_ws": "# header comment\n\n  DETECTOR   7  extra\n\tdt\t1e-3\n t0 -2\nn0_slot +4\n"
                         "nbkg_slot 5\nmap\nfunc\n# mid\ncounts 1_000 2 3\n\x0c4 5\x0b\n",
    "crlf_and_cr": "DETECTOR 0\r\ndt 0.5\r\nt0 0\rn0_slot 1\r\nnbkg_slot 2\rmap 0\r\ncounts 1 2\r3\r\n",
    "no_trailing_newline": "DETECTOR 3\n" + HDR + "counts 9 8 7",
    "counts_replaced": "DETECTOR 0\n" + HDR + "counts 1 2 3\n4 5\ncounts 7\n8\n",
    "keys_after_counts": "DETECTOR 0\n" + HDR + "counts 1 2\n3\ndt 2.5\n4\n",
    "float_forms": "DETECTOR 0\ndt 1_0.2_5e-0_3\nt0 0\nn0_slot 0\nnbkg_slot 1\nmap 0\n"
                   "func inf -Infinity nan .5 5. +1E2\ncounts 1\n",
    "dt_nan_passes": "DETECTOR 0\ndt nan\nt0 0\nn0_slot 0\nnbkg_slot 1\nmap\ncounts 1 2\n",
    "empty_file": "",
    "only_comments": "# nothing\n\n   \n",
    "before_header": "dt 0.1\nDETECTOR 0\n",
    "before_header_continuation": "12 13\n",
    "unknown_key": "DETECTOR 0\n" + HDR + "bogus 1\ncounts 1\n",
    "continuation_before_counts": "DETECTOR 0\n" + HDR + "1 2 3\n",
    "malformed_int": "DETECTOR 0\n" + HDR + "counts 1 2 x3\n",
    "malformed_float": "DETECTOR 0\ndt 0x1p3\n",
    "malformed_underscore": "DETECTOR 0\n" + HDR + "counts 1__0\n",
    "malformed_trailing_underscore": "DETECTOR 0\n" + HDR + "counts 10_\n",
    "malformed_decimal_count": "DETECTOR 0\n" + HDR + "counts 1 2\n3.0\n",
    "detector_without_index": "DETECTOR\n",
    "detector_bad_index": "DETECTOR 1.5\n",
    "dt_without_value": "DETECTOR 0\ndt\n",
    "missing_keys": "DETECTOR 4\ndt 0.1\nmap 0\n",
    "missing_all": "DETECTOR 4\n",
    "missing_before_later_malformed": "DETECTOR 4\ndt 0.1\nDETECTOR 5\ncounts x\n",
    "malformed_before_block_end": "DETECTOR 4\ndt 0.1\ncounts x\nDETECTOR 5\n",
    "negative_count": "DETECTOR 2\n" + HDR + "counts 1 2\n3 -4 5\n",
    "negative_map": "DETECTOR 2\ndt 0.1\nt0 0\nn0_slot 0\nnbkg_slot 1\nmap 0 -1\ncounts 1\n",
    "negative_map_first_of_two": "DETECTOR 2\ndt 0.1\nt0 0\nn0_slot 0\nnbkg_slot 1\nmap 0 -1\n"
                                 "counts 1\nDETECTOR 3\n" + HDR + "counts 4\n",
    "empty_histogram": "DETECTOR 2\n" + HDR + "counts\n",
    "dt_zero": "DETECTOR 2\ndt 0.0\nt0 0\nn0_slot 0\nnbkg_slot 1\nmap 0\ncounts 1\n",
    "dt_negative_second_block": "DETECTOR 0\n" + HDR + "counts 1\nDETECTOR 1\ndt -1\nt0 0\n"
                                "n0_slot 0\nnbkg_slot 1\nmap\ncounts 1\n",
    "error_after_good_blocks": "DETECTOR 0\n" + HDR + "counts 1\n" * 3 + "DETECTOR 1\n" + HDR +
                               "counts 5 6\nzz\n",
    "huge_int_fallback": "DETECTOR 0\n" + HDR + "counts 1 99999999999999999999999\n",
    "non_ascii_fallback": "# détecteur\nDETECTOR 0\n" + HDR + "counts 1 2\n",
    "non_ascii_malformed": "DETECTOR 0\n" + HDR + "counts 1 ²\n",
    "unicode_digits": "DETECTOR 0\n" + HDR + "counts 1 ٣\n",
    "nul_byte": "DETECTOR 0\n" + HDR + "counts 1 \x002\n",
    "many_blocks": "".join(f"DETECTOR {j}\n" + HDR + "counts " + " ".join(str(k * j) for k in range(40))
                           + "\n" for j in range(30)),
}
