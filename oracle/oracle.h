/*
 * oracle.h — CPU restatement of the reference resharding path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 product, not part of it. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it. It restates, in plain C, the algorithms of /root/reference/proj/include/
 * reshard/ headers (planner) and the SPEC-only executor / verifier / oracle
 * (SPEC.md:346-426), citing file:line per function in oracle.c.
 *
 * Parity pinning: the planner half is pinned against plan dumps produced by the
 * reference headers themselves (oracle/_ref/ref_plan, built by oracle/Makefile from
 * /root/reference with the one-line D1 shim; fixtures in tests/golden/). The
 * executor half has no reference code (SPEC prose only): it is pinned by content —
 * every destination element must equal canon_value(seed, k, kind)
 * (common.hpp:77-80) — which is independent of the plan.
 * The D2 extension (over-sourced ZeRO intervals, allow_oversourced=1) is
 * "parity unpinned": the reference throws there.
 */
#ifndef RESHARD_ORACLE_H
#define RESHARD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: 0 ok, 1 plan/verification violation or internal, 2 config error */
typedef struct or_scenario or_scenario;
typedef struct or_plan or_plan;
typedef struct or_state or_state;

typedef struct {
    int kind;          /* 0 param, 1 optim, 2 grad */
    int tensor;        /* tensor index or -1 for flat payloads */
    int flat;          /* 1: [lo,hi) flat interval in d[0] */
    int nd;
    int64_t lo[4], hi[4];
    int src_rank, dst_rank, src_phys, dst_phys;
    int64_t count, bytes;
} or_transfer;

or_scenario* or_scenario_parse(const char* text, char* err, size_t errlen);
void or_scenario_free(or_scenario* s);
int or_scenario_num_tensors(const or_scenario* s);
const char* or_scenario_tensor_id(const or_scenario* s, int t);
int64_t or_scenario_total_numel(const or_scenario* s);
uint64_t or_scenario_fingerprint(const or_scenario* s);

/* Plan = plan_parameters + plan_optimizer + plan_scalars + resolve_peers.
 * Returns status; *out is NULL unless 0. */
int or_plan_build(const or_scenario* s, int allow_oversourced, or_plan** out, char* err, size_t errlen);
void or_plan_free(or_plan* p);
int64_t or_plan_num_transfers(const or_plan* p);
const or_transfer* or_plan_transfers(const or_plan* p);
int64_t or_plan_bytes_moved(const or_plan* p);
int64_t or_plan_bytes_retained(const or_plan* p);
/* reference dump format (routing.hpp:86-90), one line per transfer; malloc'd */
char* or_plan_dump(const or_plan* p);
void or_free(void* ptr);

/* Regions dump for VPS tests: per rank of src (which=0) or dst (which=1):
 * "rank R param <id> [box]" lines, "rank R optim [lo:hi]" lines (ZeRO only),
 * "rank R layout dense|expert <id> [box] lo hi" lines. malloc'd. */
char* or_regions_dump(const or_scenario* s, int which, char* err, size_t errlen);

/* Executor state: one host buffer set per virtual rank of the
 * chosen side's config, in the physical layout documented in DESIGN.md §3. */
or_state* or_state_create(const or_scenario* s, int which, int with_grads, char* err, size_t errlen);
void or_state_free(or_state* st);
int or_state_num_ranks(const or_state* st);
/* buf: 0 param, 1 master, 2 m, 3 v, 4 grad, 5 scalars */
void* or_state_buffer(or_state* st, int rank, int buf, int64_t* bytes);
/* load_state: canon payload for every owned element */
void or_state_load(or_state* st, uint64_t seed);
/* zero every buffer (a fresh destination) */
void or_state_clear(or_state* st);
/* execute, buffer mode collapsed to direct copies: every plan
 * transfer, every retained region and the scalar broadcast. nthreads>=1. */
int or_execute(const or_plan* p, const or_state* src, or_state* dst, int nthreads, char* err, size_t errlen);
/* verify_state: number of elements != canon; first violation text in err */
int64_t or_verify(const or_state* st, uint64_t seed, char* err, size_t errlen);
/* oracle_reshard: gather from src replicas, redistribute by dst layout */
int or_oracle_reshard(const or_scenario* s, const or_state* src, or_state* dst, char* err, size_t errlen);
/* 1 iff all buffers byte-identical */
int or_state_equal(const or_state* a, const or_state* b);

/* canon_value (common.hpp:77-80) */
uint64_t or_canon(uint64_t seed, int64_t element, int kind);

#ifdef __cplusplus
}
#endif
#endif
