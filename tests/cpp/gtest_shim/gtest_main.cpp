// main() of the GoogleTest shim: runs every registered TEST in order, prints
// GoogleTest-style [ RUN ] / [ OK ] / [ FAILED ] lines. Arguments
// `--skip Suite.Name` leave a test out (reported as [ SKIPPED ]).
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>

#include "gtest/gtest.h"

int main(int argc, char** argv) {
    std::set<std::string> skip;
    for (int i = 1; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], "--skip")) skip.insert(argv[++i]);
    int failed = 0, passed = 0, skipped = 0;
    for (const auto& t : gtshim::registry()) {
        if (skip.count(t.name)) {
            std::printf("[ SKIPPED  ] %s\n", t.name.c_str());
            ++skipped;
            continue;
        }
        std::printf("[ RUN      ] %s\n", t.name.c_str());
        std::fflush(stdout);
        gtshim::current_failures() = 0;
        try {
            t.body();
        } catch (const std::exception& e) {
            std::printf("uncaught exception: %s\n", e.what());
            ++gtshim::current_failures();
        }
        const bool ok = gtshim::current_failures() == 0;
        std::printf("%s %s\n", ok ? "[       OK ]" : "[  FAILED  ]", t.name.c_str());
        (ok ? passed : failed)++;
    }
    std::printf("[==========] %d passed, %d failed, %d skipped\n", passed, failed, skipped);
    return failed ? 1 : 0;
}
