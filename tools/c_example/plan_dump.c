/* A plain-C caller of the drop-in boundary (include/reshard_b200.h): reads a scenario
 * file, builds the plan (host planner, or the GPU planner with --gpu), prints the
 * reference dump format and the summary. What a cgo / JNI / N-API binding would call.
 *
 *   cc -O2 -I include tools/c_example/plan_dump.c -L paper_2605_18815_b200/_lib \
 *      -lreshard_b200 -Wl,-rpath,$PWD/paper_2605_18815_b200/_lib -o plan_dump
 *   ./plan_dump scenario.txt [--gpu]
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "reshard_b200.h"

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s <scenario> [--gpu]\n", argv[0]);
        return 2;
    }
    FILE* f = fopen(argv[1], "rb");
    if (!f) {
        perror(argv[1]);
        return 2;
    }
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    char* text = malloc((size_t)n + 1);
    if (fread(text, 1, (size_t)n, f) != (size_t)n) {
        fclose(f);
        return 2;
    }
    text[n] = 0;
    fclose(f);
    rs_plan_t* plan = NULL;
    int rc = rs_plan_from_scenario(text, 0, &plan);
    free(text);
    if (rc != RS_OK) {
        /* the reference CLI maps ConfigError to exit code 2 */
        printf("# error: %s\n", rs_last_error());
        return rc == RS_ERR_CONFIG ? 2 : 1;
    }
    char* dump = NULL;
    size_t len = 0;
    rc = rs_plan_dump(plan, (argc > 2 && !strcmp(argv[2], "--gpu")) ? 0 : -1, &dump, &len);
    if (rc != RS_OK) {
        fprintf(stderr, "dump failed: %s\n", rs_last_error());
        rs_plan_destroy(plan);
        return 1;
    }
    fwrite(dump, 1, len, stdout);
    rs_free(dump);
    rs_plan_summary_t s;
    rs_plan_summary(plan, &s);
    printf("# transfers=%lld bytes_moved=%lld bytes_retained=%lld\n", (long long)s.num_transfers,
           (long long)s.bytes_moved, (long long)s.bytes_retained);
    rs_plan_destroy(plan);
    return 0;
}
