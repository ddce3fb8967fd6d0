/*
 * sm2batch.h -- drop-in header name for consumers of the reference library.
 *
 * Code written against the reference's <sm2batch.h> (its enum sm2b_status 0..7, the opaque
 * sm2b_ctx, sm2b_op_counts, sm2b_bench_report and the twelve sm2b_* entry points,
 * /root/reference/proj/include/sm2batch.h:27-105) compiles unchanged with -I<this directory>
 * and links against libgecc_b200.so instead of libsm2batch.so.  The declarations themselves live
 * in gecc_b200.h, Part 1 (each one cites the reference line it replaces); Part 2 of that header
 * (gecc_*: curve selector, column-buffer batch API, MSM, device-pointer forms, group contexts)
 * comes along and does not collide with anything the reference declares.
 *
 * tests/test_abi.py::test_sm2batch_h_is_a_drop_in compiles a C translation unit that uses only
 * this header and checks the struct layouts (sizeof / offsetof) against the reference's.
 */
#ifndef SM2BATCH_H
#define SM2BATCH_H
#include "gecc_b200.h"
#endif /* SM2BATCH_H */
